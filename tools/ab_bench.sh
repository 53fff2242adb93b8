# bench.py A/B of library variants, alternating order: bash tools/ab_bench.sh rounds variant...
rounds=$1; shift
for r in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" != cur ]; then export GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_$v.so; else unset GEMMGUARD_LIB; fi
    timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('$v', round(d['value'], 1), round(d['unprotected_tflops'], 1), round(d['overhead_pct'], 2), round(d['e2e']['value'], 1), d['clocks']['sm_mhz'])"
  done
  set -- $(printf '%s\n' "$@" | tac)
done
unset GEMMGUARD_LIB
