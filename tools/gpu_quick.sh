# quick GPU iteration: new-kernel tests + bench (no cpu baseline, short e2e)
set -x
timeout 600 python -m pytest tests -m gpu -x -q  2>&1 | tail -8
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -3 gpurun_out/bench_q.err
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print(d['ms_per_step'],d['roofline']);[print(k,v) for k,v in d['kernels'].items()]"
