# quick GPU iteration: gpu tests + bench (no cpu baseline, short e2e); usage: bash tools/gpu_quick.sh [pytest -k expr]
set -x
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 600 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -15;
else timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; fi
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -3 gpurun_out/bench_q.err
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print(d['ms_per_step'],d['value'],d['roofline']);[print(k,v) for k,v in d['kernels'].items()];print('e2e',d['e2e'])"
