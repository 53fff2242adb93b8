"""Protected vs unprotected timing of one shape with SM-clock / power samples (pynvml) taken during
a ~1.5 s loop of each; GG_DEBUG selects the diagnostic switches (read once per process)."""
import os, sys, threading, time, torch
import pynvml
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in sys.argv[1:4]]
dt = {'bf16': torch.bfloat16, 'f16': torch.float16, 'tf32': torch.float32}[sys.argv[4] if len(sys.argv) > 4 else 'bf16']
x = torch.randn(M, Kd, device='cuda').to(dt); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(dt)
b = torch.zeros(N, device='cuda')
ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, dt); bsv = bs.item()
y = torch.empty(M, N, dtype=K.default_out_dtype(dt), device='cuda'); res = K.CheckResult.empty(M, False, 'cuda')
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def t(fn):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    t0 = time.time(); n = 0
    while time.time() - t0 < 0.3: fn(); n += 1
    torch.cuda.synchronize()
    iters = max(20, int(n * 1.5 / 0.3))
    samples = []; stop = [False]
    def samp():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
            time.sleep(0.05)
    th = threading.Thread(target=samp); th.start()
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize(); stop[0] = True; th.join()
    samples = sorted(samples[2:-1] or samples)
    mid = samples[len(samples) // 2]
    return s.elapsed_time(e) / iters * 1e3, mid[0], sum(p for _, p in samples) / len(samples)
tu, cu, pu = t(lambda: K.protected_gemm(x, w, b, protect=False, out=y))
tp, cp, pp = t(lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y, result=res))
print(f"GG_DEBUG={os.environ.get('GG_DEBUG', '0'):>2} {M}x{N}x{Kd}: unprot {tu:7.1f}us {cu}MHz {pu:5.0f}W | prot {tp:7.1f}us {cp}MHz {pp:5.0f}W | overhead {100*(tp/tu-1):5.1f}% cycles-overhead {100*(tp*cp/(tu*cu)-1):5.1f}%", flush=True)
