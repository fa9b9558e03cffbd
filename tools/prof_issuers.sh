# Source-level ncu captures of the headline layer's kernels (fwd_factored, bwd_fused) and the
# one-pass stream backward, to read the producer / MMA-issuer warps' instruction counts and stalls.
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fwd_factored|bwd_fused" -s 2 -c 2 \
  -o gpurun_out/pi_layer python tools/prof_layer.py 3 > gpurun_out/pi_layer.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bwd_onepass" -c 1 \
  -o gpurun_out/pi_op python tools/prof_stream.py 4096 1 > gpurun_out/pi_op.log 2>&1
for r in pi_layer pi_op; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_src.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out/pi_*
