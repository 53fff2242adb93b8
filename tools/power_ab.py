"""Interleaved sustained A/B under the power cap: cuBLAS (torch.matmul) vs our unprotected vs
protected launches of one shape; each arm runs ~1 s per round, 3 rounds, reporting time per launch,
median SM clock and mean power (pynvml).  Usage: power_ab.py M N K [seconds]"""
import sys, threading, time, torch
import pynvml
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in sys.argv[1:4]]
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
x = torch.randn(M, Kd, device='cuda').to(torch.bfloat16); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(torch.bfloat16)
b = torch.zeros(N, device='cuda')
ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, torch.bfloat16); bsv = bs.item()
y = torch.empty(M, N, dtype=torch.bfloat16, device='cuda'); res = K.CheckResult.empty(M, False, 'cuda')
bb = b.to(torch.bfloat16)
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
arms = {
    'cublas': lambda: torch.addmm(bb, x, w.t(), out=y),
    'unprot': lambda: K.protected_gemm(x, w, b, protect=False, out=y),
    'prot': lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y, result=res),
}
def run(fn):
    torch.cuda.synchronize(); t0 = time.time(); n = 0
    while time.time() - t0 < 0.1: fn(); n += 1
    torch.cuda.synchronize()
    iters = max(10, int(n * secs / 0.1))
    samples = []; stop = [False]
    def samp():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
            time.sleep(0.02)
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    th = threading.Thread(target=samp); th.start(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize(); stop[0] = True; th.join()
    sm = sorted(samples[len(samples) // 4:]) or samples
    return s.elapsed_time(e) / iters * 1e3, sm[len(sm) // 2][0], sum(p for _, p in sm) / len(sm)
for fn in arms.values():
    for _ in range(3): fn()
res_ = {k: [] for k in arms}
for rnd in range(3):
    for k, fn in arms.items():
        res_[k].append(run(fn))
fl = 2 * M * N * Kd
out = []
for k, v in res_.items():
    t = sorted(r[0] for r in v)[1]
    out.append(f"{k} {t:8.1f}us {fl / t / 1e6:6.0f}TF {sorted(r[1] for r in v)[1]:5d}MHz {sum(r[2] for r in v) / 3:4.0f}W")
print(f"{M}x{N}x{Kd}: " + " | ".join(out), flush=True)
