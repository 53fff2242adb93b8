"""Dump per-tile predicted/observed partials from the workspace vs CPU expectations."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
BM, BN = 128, 256

def ws_offsets(M, N):
    mt = (M + BM - 1) // BM; nt = (N + BN - 1) // BN; mp = mt * BM
    al = lambda v: (v + 255) // 256 * 256
    off = 0; o = {}
    o['counters'] = off; off = al(off + 16)
    o['band_counter'] = off; off = al(off + 4 * mt)
    o['band_active'] = off; off = al(off + mt)
    o['band_nflag'] = off; off = al(off + 4 * mt)
    o['band_maxkey'] = off; off = al(off + 8 * mt)
    o['pred'] = off; off = al(off + 8 * mp * nt)
    o['partial'] = off; off = al(off + 8 * mp * nt)
    return o, mt, nt, mp

for (M, N, Kd) in [(517, 1000, 3072), (517, 1000, 768), (517, 768, 3072), (128, 1024, 3072), (256, 1024, 512), (197, 768, 768)]:
    g = torch.Generator().manual_seed(1)
    x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8).cuda()
    w = torch.randint(-128, 128, (N, Kd), generator=g, dtype=torch.int8).cuda()
    b = torch.randint(-64, 65, (N,), generator=g, dtype=torch.int32).cuda()
    ws_, bs = K.offline_checksum(w, b, L.GG_P_I64)
    y, res = K.protected_gemm(x, w, b, w_sum=ws_, bias_sum=bs.item())
    torch.cuda.synchronize()
    work = K.workspace(M, N, x.device)
    o, mt, nt, mp = ws_offsets(M, N)
    pred = work[o['pred']:o['pred'] + 8 * mp * nt].view(torch.int64).view(nt, mp).cpu()
    part = work[o['partial']:o['partial'] + 8 * mp * nt].view(torch.int64).view(nt, mp).cpu()
    xc, wc, yc = x.cpu().long(), ws_.cpu(), y.cpu().long()
    kb_n = 128
    kblocks = (Kd + kb_n - 1) // kb_n
    bad_pred = bad_obs = 0
    for n in range(nt):
        ks = [k for kb in range(kblocks) if kb % nt == n for k in range(kb * kb_n, min(Kd, kb * kb_n + kb_n))]
        ep = (xc[:, ks] @ wc[ks]) if ks else torch.zeros(M, dtype=torch.int64)
        eo = yc[:, n * BN:min(N, n * BN + BN)].sum(1)
        bp = torch.nonzero(pred[n, :M] != ep).flatten(); bo = torch.nonzero(part[n, :M] != eo).flatten()
        bad_pred += bp.numel(); bad_obs += bo.numel()
        if bp.numel(): print(f'  {M}x{N}x{Kd} tile n={n}: pred bad rows {bp.numel()} first {bp[:6].tolist()} got {pred[n, bp[:3]].tolist()} want {ep[bp[:3]].tolist()}')
        if bo.numel(): print(f'  {M}x{N}x{Kd} tile n={n}: obs bad rows {bo.numel()} first {bo[:6].tolist()}')
    dref = (xc @ wc + int(bs.item())) - yc.sum(1)
    print(f'{M}x{N}x{Kd}: bad pred {bad_pred} bad obs {bad_obs} bad d {(res.d.cpu() != dref).sum().item()}', flush=True)
