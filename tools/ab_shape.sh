# A/B of library variants on one shape, alternating the run order: bash tools/ab_shape.sh "M N K" rounds variant...
shape=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" != cur ]; then export GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_$v.so; else unset GEMMGUARD_LIB; fi
    echo -n "[$v] "; timeout 60 python tools/dbg_perf.py $shape
  done
  set -- $(printf '%s\n' "$@" | tac)
done
unset GEMMGUARD_LIB
