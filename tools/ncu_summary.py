"""Summarise an .ncu-rep: key metrics per kernel + SASS hot regions."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__cycles_elapsed.avg']
for r in rows[2:]:
    print('---', r[hdr.index('Kernel Name')][:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w); print(f'  {w:70s} {r[i]} {units[i]}')
if len(sys.argv) > 2:
    k = int(sys.argv[2])
    s = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--launch-skip', str(k), '--launch-count', '1',
                        '--print-source', 'sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(s)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith('0x')]
    ii = hdr.index('Instructions Executed'); si = hdr.index('Warp Stall Sampling (All Samples)')
    tot = sum(float(r[ii] or 0) for r in data); tots = sum(float(r[si] or 0) for r in data)
    print('total inst', tot, 'samples', tots)
    W = 80
    for s0 in range(0, len(data), W):
        c = sum(float(r[ii] or 0) for r in data[s0:s0 + W]); st = sum(float(r[si] or 0) for r in data[s0:s0 + W])
        if c / tot > 0.01 or st / tots > 0.01:
            ops = {}
            for r in data[s0:s0 + W]:
                t = r[1].split()
                op = t[1] if t and t[0].startswith('@') else (t[0] if t else '')
                ops[op] = ops.get(op, 0) + float(r[ii] or 0)
            top = sorted(ops.items(), key=lambda x: -x[1])[:7]
            print(f"{s0:5d} inst {c / tot * 100:5.1f}% stall {st / tots * 100:5.1f}% | " + ", ".join(f"{k}:{v / 1e6:.2f}M" for k, v in top))
