# ncu --set full of one kernel family (regex $1) on tools/prof_layer.py; report name $2
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -s 2 -c 2 -o gpurun_out/$2 python tools/prof_layer.py 3 > gpurun_out/$2.log 2>&1
tail -3 gpurun_out/$2.log
