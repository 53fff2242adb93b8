"""Quick kernel timing probe (CUDA events, L2-flushed between iterations)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L

def t(fn, iters=20, warm=3):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
    for _ in range(warm): fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts)//2]

for dt in [torch.bfloat16, torch.int8, torch.float16, torch.float32]:
    for (M,N,Kd) in [(50432,2304,768),(50432,768,768),(50432,3072,768),(50432,768,3072),(8192,8192,8192),(197,768,768)]:
        if dt==torch.int8:
            x=torch.randint(-128,128,(M,Kd),dtype=torch.int8,device='cuda'); w=torch.randint(-128,128,(N,Kd),dtype=torch.int8,device='cuda'); b=torch.zeros(N,dtype=torch.int32,device='cuda')
            prec=L.GG_P_I64
        else:
            x=torch.randn(M,Kd,device='cuda').to(dt); w=(torch.randn(N,Kd,device='cuda')/Kd**.5).to(dt); b=torch.zeros(N,device='cuda')
            prec=L.GG_P_F64
        ws,bs=K.offline_checksum(w,b,prec); aux=K.checksum_aux(ws,dt)
        y=torch.empty(M,N,dtype=K.default_out_dtype(dt),device='cuda')
        res=K.CheckResult.empty(M,dt==torch.int8,'cuda')
        tu=t(lambda: K.protected_gemm(x,w,b,protect=False,out=y))
        bsv=bs.item(); tp=t(lambda: K.protected_gemm(x,w,b,w_sum=ws,w_aux=aux,bias_sum=bsv,lo=-1e30,hi=1e30,out=y,result=res))
        fl=2*M*N*Kd
        ref=None
        if dt!=torch.int8:
            ref=t(lambda: torch.matmul(x,w.T))
        print(f"{str(dt):15s} {M}x{N}x{Kd}: unprot {tu*1e3:8.1f}us {fl/tu/1e9:7.1f} TF | prot {tp*1e3:8.1f}us {fl/tp/1e9:7.1f} TF overhead {100*(tp/tu-1):5.2f}% | torch {'' if ref is None else f'{fl/ref/1e9:.1f} TF'}", flush=True)
