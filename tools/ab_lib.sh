# A/B of two builds: the saved baseline (librsa_b200_base.so) against the current library.
# bench.py (headline), long_kernels.py 8192 (both modes, per kernel).  Output under gpurun_out/.
mkdir -p gpurun_out
for lib in base cur; do
  if [ $lib = base ]; then export RSA_B200_LIB=$PWD/paper_2105_13120_b200/librsa_b200_base.so; else unset RSA_B200_LIB; fi
  timeout 600 python bench.py > gpurun_out/ab_bench_$lib.json 2> gpurun_out/ab_bench_$lib.err
  timeout 300 python tools/long_kernels.py 8192 > gpurun_out/ab_lk_$lib.txt 2>&1
done
unset RSA_B200_LIB
python - <<'PY'
import json
for lib in ("base", "cur"):
    b = json.loads(open(f"gpurun_out/ab_bench_{lib}.json").read().strip().splitlines()[-1])
    lk = json.loads(open(f"gpurun_out/ab_lk_{lib}.txt").read().strip().splitlines()[-1])
    ks = {m: {k: v["us"] for k, v in lk[m]["kernels"].items()} for m in ("panel", "stream")}
    print(lib, "bench ms/step", b["ms_per_step"], "roofline", b["roofline"]["frac"], ks)
PY
