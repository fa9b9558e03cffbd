# round-2 profile evidence: launch list of the bench (ncu gpu__time_duration), one --set full
# capture of the bench layer's kernels, and the traffic of the dominant kernel
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/b_ncu_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fwd_|bwd_|rowdot" -s 3 -c 3 \
  -o gpurun_out/prof_$TAG python tools/prof_layer.py 3 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
