# A/B timing of library variants in one box: bash tools/ab.sh lib1 lib2 ...  (paths under paper_2105_13120_b200/)
for round in 1 2; do
  for v in "$@"; do
    r=$(RSA_B200_LIB=paper_2105_13120_b200/$v timeout 60 python tools/ff_exp.py 0 0 2>&1 | tail -1)
    echo "$v $r"
  done
done
