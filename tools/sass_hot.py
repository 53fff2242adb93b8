"""Top stalled / most-executed SASS instructions of one launch in an .ncu-rep.

    python tools/sass_hot.py REP LAUNCH_INDEX [N]
"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--launch-skip', str(k), '--launch-count', '1',
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r)
h, data = rows[hi], [r for r in rows[hi + 1:] if len(r) == len(rows[hi]) and r[0].startswith('0x')]
S = h.index('Warp Stall Sampling (All Samples)'); E = h.index('Instructions Executed')
stalls = [c for c in h if c.startswith('stall_') and '(Not' not in c]
tot = sum(float(r[S] or 0) for r in data) or 1
tote = sum(float(r[E] or 0) for r in data) or 1
print(f'total samples {tot:.0f}  instructions {tote:.3g}')
for i, r in sorted(enumerate(data), key=lambda x: -float(x[1][S] or 0))[:n]:
    top = sorted(((c[6:], float(r[h.index(c)] or 0)) for c in stalls), key=lambda x: -x[1])[:3]
    print(f'{i:5d} {100*float(r[S] or 0)/tot:5.1f}% ex={float(r[E] or 0):9.0f} {r[1][:60]:60s} ' +
          ' '.join(f'{a}:{b:.0f}' for a, b in top if b))
