mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bwd_onepass" -c 1 -o gpurun_out/prof_fs python tools/prof_stream.py 4096 1 > gpurun_out/prof_fs.log 2>&1
tail -3 gpurun_out/prof_fs.log
ncu -i gpurun_out/prof_fs.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_fs_src.csv 2>/dev/null
ncu -i gpurun_out/prof_fs.ncu-rep --page raw --csv > gpurun_out/prof_fs_raw.csv 2>/dev/null
python tools/sass_stalls.py gpurun_out/prof_fs_src.csv 40
