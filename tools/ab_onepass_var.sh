# One-pass backward variants (tools/build_all_variant.sh NAME "-D..."): long_kernels 8192 per
# library, then the one-pass parity tests on the last one.  usage: bash tools/ab_onepass_var.sh cur NAME ...
for lib in "$@"; do
  if [ $lib = cur ]; then unset RSA_B200_LIB; else export RSA_B200_LIB=$PWD/paper_2105_13120_b200/librsa_b200_$lib.so; fi
  timeout 300 python tools/long_kernels.py 8192 2>/dev/null | tail -n 1 | python -c "
import json,sys; lk=json.loads(sys.stdin.read()); print('$lib', {m: {k: v['us'] for k, v in lk[m]['kernels'].items() if k != 'rowdot'} for m in ('panel','stream')})"
done
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_panel_onepass.py -x -q 2>&1 | tail -n 1
