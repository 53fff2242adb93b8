"""Stall samples of every mbarrier wait loop of one launch, grouped by barrier offset.

    python tools/sass_waits.py REP LAUNCH_INDEX
"""
import csv, io, re, subprocess, sys
rep, k = sys.argv[1], int(sys.argv[2])
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--launch-skip', str(k), '--launch-count', '1',
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith('0x')]
data = data[:len(data) // 2] if len(data) % 2 == 0 and data[:len(data)//2] == data[len(data)//2:] else data
S, E = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
tot = sum(float(r[S] or 0) for r in data)
agg = {}
for i, r in enumerate(data):
    m = re.search(r'TRYWAIT\S* P\d, \[R\d+\+URZ(?:\+(0x[0-9a-f]+))?\]', r[1])
    if not m:
        continue
    off = m.group(1) or '0x0'
    s = sum(float(data[j][S] or 0) for j in range(i - 1, min(i + 4, len(data))))
    a = agg.setdefault(off, [0.0, 0.0])
    a[0] += s
    a[1] += float(r[E] or 0)
for off, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f'{off:>8s}  stall {100*s/tot:5.1f}%  tries {e:10.0f}')
