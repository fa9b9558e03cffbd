# A/B of the one-pass backwards: the saved baseline library (librsa_b200_base.so) against the
# current build, at L = 8192 (stream: tools/fs_exp.py; both modes: tools/long_kernels.py),
# then the one-pass parity tests.  Output under gpurun_out/.
mkdir -p gpurun_out
for lib in base cur; do
  if [ $lib = base ]; then export RSA_B200_LIB=$PWD/paper_2105_13120_b200/librsa_b200_base.so; else unset RSA_B200_LIB; fi
  timeout 180 python tools/fs_exp.py 8192 > gpurun_out/ab_fs_$lib.txt 2>&1
  timeout 300 python tools/long_kernels.py 8192 > gpurun_out/ab_lk_$lib.txt 2>&1
done
unset RSA_B200_LIB
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_panel_onepass.py -x -q > gpurun_out/ab_tests.txt 2>&1
tail -3 gpurun_out/ab_*.txt
