# full round evidence: gpu tests, smoke, bench, launch list, ncu --set full of the fused kernels
# usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r1}
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_ncu_$TAG.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fwd_|bwd_|rowdot" -s 3 -c 3 -o gpurun_out/prof_$TAG python tools/prof_layer.py 3 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
