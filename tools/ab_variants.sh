# A/B timing of library variants (tools/dbg_perf.py per shape) + traces; usage: bash tools/ab_variants.sh [variant ...]
for s in "50432 3072 768" "50432 768 768" "50432 768 3072" "50432 2304 768"; do
  for v in "" "$@"; do
    if [ -n "$v" ]; then export GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_$v.so; else unset GEMMGUARD_LIB; fi
    echo -n "[$v] "; timeout 60 python tools/dbg_perf.py $s
  done
done
unset GEMMGUARD_LIB
