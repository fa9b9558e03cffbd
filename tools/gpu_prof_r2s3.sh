# round-2 (session 3) profile evidence: ncu --set full of the one-pass backward kernels
# (stream and panel instantiations) at L = 4096, their summaries, configs 1/4/5 and the bench
TAG=${1:-r2s3}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bwd_onepass" -c 2 \
  -o gpurun_out/prof_onepass_$TAG sh -c "python tools/prof_stream.py 4096 1 && python tools/prof_long.py 4096" \
  > gpurun_out/ncu_onepass_$TAG.log 2>&1
tail -2 gpurun_out/ncu_onepass_$TAG.log
ncu -i gpurun_out/prof_onepass_$TAG.ncu-rep --page raw --csv > gpurun_out/onepass_raw_$TAG.csv 2>/dev/null
timeout 900 python tools/configs.py > gpurun_out/configs_$TAG.json 2> gpurun_out/configs_$TAG.err
tail -c 600 gpurun_out/configs_$TAG.json
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['roofline']['step']['frac'],d['parity']['pass'],d['e2e']['value'])"
