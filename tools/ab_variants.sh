# Forward variants (built by tools/build_all_variant.sh NAME): long_kernels.py 8192 and bench.py
# per library.  usage: bash tools/ab_variants.sh cur poly3 poly4
mkdir -p gpurun_out
for lib in "$@"; do
  if [ $lib = cur ]; then unset RSA_B200_LIB; else export RSA_B200_LIB=$PWD/paper_2105_13120_b200/librsa_b200_$lib.so; fi
  lk=$(timeout 300 python tools/long_kernels.py 8192 2>/dev/null | tail -n 1)
  bj=$(timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -n 1)
  python - "$lib" "$lk" "$bj" <<'PY'
import json, sys
lib, lk, bj = sys.argv[1], json.loads(sys.argv[2]), json.loads(sys.argv[3])
print(lib, "L8192", {m: {k: v["us"] for k, v in lk[m]["kernels"].items() if k != "rowdot"} for m in ("panel", "stream")},
      "bench", round(bj["ms_per_step"], 4), {k: round(v["us_per_launch"], 1) for k, v in bj["kernels"].items()},
      "parity", bj.get("parity", {}).get("pass"))
PY
done
