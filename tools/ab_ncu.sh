# Locked-clock (ncu base clocks) A/B of library variants: per-launch kernel durations of
# tools/prof_one.py (2 unprotected + 2 protected launches) per shape.
# usage: bash tools/ab_ncu.sh "M N K" variant...   (variant "cur" = the in-tree library)
shape=$1; shift
for v in "$@"; do
  if [ "$v" != cur ]; then export GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_$v.so; else unset GEMMGUARD_LIB; fi
  ncu --metrics gpu__time_duration.sum -k regex:gg_protected --csv python tools/prof_one.py $shape ${DT:-bf16} 2>/dev/null \
    | python -c "
import sys, csv
rows = list(csv.reader(sys.stdin)); h = next(r for r in rows if 'Kernel Name' in r); K = h.index('Kernel Name'); V = h.index('Metric Value')
import re
prot = lambda r: re.search(r'pair_kernel<\\d+, \\d+, (\\d)', r[K]).group(1) == '1'  # <KIND, OUT, PROTECT, CLAIM>
body = [r for r in rows[rows.index(h) + 1:] if len(r) == len(h) and 'pair_kernel<' in r[K]]
u = [float(r[V].replace(',', '')) for r in body if not prot(r)]
p = [float(r[V].replace(',', '')) for r in body if prot(r)]
print(f'[$v] $shape unprot {sum(u)/len(u)/1e3:.1f}us prot {sum(p)/len(p)/1e3:.1f}us overhead {100*(sum(p)/len(p)/(sum(u)/len(u))-1):.1f}%')
"
done
unset GEMMGUARD_LIB
