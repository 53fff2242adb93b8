"""Per-tile role timeline of one protected GEMM from the GG_TRACE library.

    GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_trace.so \
        python tools/trace_tiles.py M N K [protect] [bf16|f16|tf32]
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in sys.argv[1:4]]
protect = (sys.argv[4] != '0') if len(sys.argv) > 4 else True
dt = {'bf16': torch.bfloat16, 'f16': torch.float16, 'tf32': torch.float32}[sys.argv[5] if len(sys.argv) > 5 else 'bf16']
x = torch.randn(M, Kd, device='cuda').to(dt); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(dt)
b = torch.zeros(N, device='cuda')
ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, dt); bsv = bs.item()
y = torch.empty(M, N, dtype=K.default_out_dtype(dt), device='cuda'); res = K.CheckResult.empty(M, False, 'cuda')
lib = L.load(); lib.gg_trace_buffer.argtypes = [ctypes.c_void_p]
TT, EV = 64, 28
buf = torch.zeros(148 * TT * EV + 4 * 64 * 4, dtype=torch.int64, device='cuda')
act = int(os.environ.get('ACT', '0'))  # 1: the fused tanh-GELU epilogue
run = (lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y, result=res,
                                act=act)) \
    if protect else (lambda: K.protected_gemm(x, w, b, protect=False, out=y, act=act))
for _ in range(3): run()
torch.cuda.synchronize()
lib.gg_trace_buffer(ctypes.c_void_p(buf.data_ptr()))
run(); torch.cuda.synchronize()
lib.gg_trace_buffer(ctypes.c_void_p(0))
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:148 * TT * EV].reshape(148, TT, EV)
det = allb[148 * TT * EV:].reshape(4, 64, 4)
if os.environ.get('DETAIL'):
    c = 0
    base = det[c][det[c] > 0].min() if (det[c] > 0).any() else 0
    for kb in range(64):
        r = det[c, kb]
        if r[3] or r[0]:
            f = lambda v: v - base if v else -1
            print(f' kb {kb:2d}: mma full-ok/relay {f(r[3]):7d} | chk wait start {f(r[0]):7d} end {f(r[1]):7d} copy end {f(r[2]):7d}')
names = {0: 'epi_tfull', 1: 'epi_tmem_rel', 2: 'epi_done', 3: 'epi_slot', 4: 'mma_start', 5: 'mma_end',
         6: 'chk_done', 7: 'chk_slot', 8: 'red_got', 9: 'red_done', 10: 'mma_wait_tempty', 11: 'red_wait', 12: 'red_obs'}
def stats(cta):
    r = t[cta]; n = int((r[:, 4] > 0).sum()) if cta % 2 == 0 else int((r[:, 0] > 0).sum())
    return r, n
for cta in (0, 1, 40, 41):
    r, n = stats(cta)
    base = r[r > 0].min() if (r > 0).any() else 0
    print(f'--- CTA {cta}: tiles {n}')
    for i in range(min(n, 12)):
        row = r[i]
        f = lambda e: (row[e] - base) if row[e] > 0 else -1
        print(f' tile {i:2d}: mma wait {f(10):8d} start {f(4):8d} end {f(5):8d} | epi tfull {f(0):8d} rel {f(1):8d} done {f(2):8d} slot {f(3):8d}'
              f' | chk done {f(6):8d} slot {f(7):8d} | red wait {f(11):8d} obs {f(12):8d} got {f(8):8d} done {f(9):8d}')
# aggregate over leader CTAs: mma issue time vs epilogue time per tile
mma, epi, gapt = [], [], []
for cta in range(0, 148, 2):
    r, n = stats(cta)
    for i in range(1, min(n, TT)):
        if r[i, 4] and r[i, 5]: mma.append(r[i, 5] - r[i, 4])
        if r[i, 0] and r[i, 2]: epi.append(r[i, 2] - r[i, 0])
        if r[i, 4] and r[i, 10]: gapt.append(r[i, 4] - r[i, 10])
ld = [t[c, i, 13] for c in range(148) for i in range(TT) if t[c, i, 0] > 0]
cp = [t[c, i, 14] for c in range(148) for i in range(TT) if t[c, i, 0] > 0]
st = [t[c, i, 15] for c in range(148) for i in range(TT) if t[c, i, 0] > 0]
ob = [t[c, i, 16] for c in range(148) for i in range(TT) if t[c, i, 0] > 0]
print('epilogue per tile (median cycles): tmem load+wait', np.median(ld), 'convert', np.median(cp), 'obs', np.median(ob), 'stage+tma', np.median(st))
pe = [t[c, i, 17] for c in range(148) for i in range(TT) if t[c, i, 17] > 0]
pc = [t[c, i, 18] for c in range(0, 148) for i in range(TT) if t[c, i, 17] > 0]
mf = [t[c, i, 19] for c in range(0, 148, 2) for i in range(TT) if t[c, i, 4] > 0]
print('per tile (median cycles): producer wait empty', np.median(pe) if pe else None, 'producer wait chkdone',
      np.median(pc) if pc else None, 'mma wait full', np.median(mf) if mf else None)
cw = [t[c, i, 20] for c in range(148) for i in range(TT) if t[c, i, 6] > 0]
cc = [t[c, i, 21] for c in range(148) for i in range(TT) if t[c, i, 6] > 0]
cm = [t[c, i, 22] for c in range(148) for i in range(TT) if t[c, i, 6] > 0]
cu = [t[c, i, 23] for c in range(148) for i in range(TT) if t[c, i, 6] > 0]
if cw: print('checksum warps per tile (median cycles): wait aready', np.median(cw), 'copy(lds)', np.median(cc), 'fence+arrive', np.median(cm), 'compute', np.median(cu))
print('median cycles: mma issue', np.median(mma) if mma else None, 'epilogue', np.median(epi) if epi else None,
      'mma wait tempty', np.median(gapt) if gapt else None)
# tail: per CTA, reducer done minus epilogue done on the CTA's last tile, and per-tile reducer latency
tails, lat = [], []
for cta in range(148):
    r = t[cta]
    idx = [i for i in range(TT) if r[i, 2] > 0 and r[i, 9] > 0]
    if not idx: continue
    i = idx[-1]
    tails.append(r[i, 9] - r[i, 2])
    lat += [r[j, 9] - r[j, 8] for j in idx]
if tails:
    print('reducer tail after last epilogue (cycles): median', np.median(tails), 'max', np.max(tails),
          '| reducer per-tile work (got->done): median', np.median(lat), 'p90', np.percentile(lat, 90), 'max', np.max(lat))

# last band finish of each CTA (overwritten per finish): compute / atomics / stores
fc = [(t[c, 0, 25] - t[c, 0, 24], t[c, 0, 26] - t[c, 0, 25], t[c, 0, 27] - t[c, 0, 26]) for c in range(148) if t[c, 0, 24] > 0]
if fc:
    a = np.array(fc)
    print('last band finish (median cycles): d/flags compute', np.median(a[:, 0]), 'summary atomics', np.median(a[:, 1]),
          'row stores', np.median(a[:, 2]))

# the CTA with the longest reducer tail: its last tiles, relative to that tile's epilogue end
if tails:
    worst = [c for c in range(148) if any(t[c, i, 2] > 0 and t[c, i, 9] > 0 for i in range(TT))]
    wc = worst[int(np.argmax(tails))]
    r = t[wc]
    idx = [i for i in range(TT) if r[i, 2] > 0 and r[i, 9] > 0]
    ref = r[idx[-1], 2]
    print(f'worst tail: CTA {wc}, tiles {len(idx)}; events relative to its last epilogue end')
    for i in idx[-4:]:
        f = lambda e: int(r[i, e] - ref) if r[i, e] > 0 else None
        print(f'  tile {i:2d}: epi done {f(2)} | chk done {f(6)} slot {f(7)} | red wait {f(11)} obs {f(12)} got {f(8)} done {f(9)}')

# per-CTA span (one SM clock each): first event to the last reducer / epilogue event
spans = []
for cta in range(148):
    r = t[cta]
    ev = r[:, :13][r[:, :13] > 0]
    if ev.size: spans.append((int(ev.max() - ev.min()), cta, int((r[:, 0] > 0).sum())))
if spans:
    s = sorted(spans)
    print('per-CTA span (cycles): min', s[0], 'median', s[len(s) // 2], 'max', s[-1])
    print('  longest 6:', s[-6:])
