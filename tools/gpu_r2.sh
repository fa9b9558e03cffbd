# round-2 GPU iteration: selected tests, full gpu suite, bench; usage: bash tools/gpu_r2.sh <tag> [pytest -k expr]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$2" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$2" 2>&1 | tail -25 > gpurun_out/tests_$TAG.txt;
else timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/tests_$TAG.txt; fi
cat gpurun_out/tests_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print(d["ms_per_step"], d["value"], json.dumps(d["roofline"]))
for k, v in d["kernels"].items(): print(k, v)
print("sum/step", d["kernel_sum_over_step"], "parity", d["parity"])
print("e2e", d["e2e"]["value"], "cpu", d.get("cpu_baseline", {}).get("value"))
PY
