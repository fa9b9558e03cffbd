for round in 1 2; do
  for v in "$@"; do
    f=$(RSA_B200_LIB=paper_2105_13120_b200/$v timeout 60 python tools/ff_exp.py 0 2>&1 | grep dbg)
    b=$(RSA_B200_LIB=paper_2105_13120_b200/$v BF_TRACE_OUT=/tmp/x.bin timeout 60 python tools/ff_exp.py 2>&1 | grep bwd)
    echo "$v $f | $b"
  done
done
