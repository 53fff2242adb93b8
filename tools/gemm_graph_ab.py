"""GEMM-only step graph (the 50 ViT-B/16 b256 GEMMs on distinct buffers), protected vs unprotected
vs cuBLAS, alternating rounds — bench.py's gemm_only — for A/B of library variants ($GEMMGUARD_LIB)."""
import os, sys, types, torch
sys.path.insert(0, '.')
import bench
args = types.SimpleNamespace(steps=20, warmup=5)
dev = torch.device('cuda', 0)
out = bench.gemm_only(args, dev, 1, torch.cuda.current_stream(dev))
print(os.environ.get('GEMMGUARD_LIB', 'default').split('/')[-1],
      {k: round(v, 2) for k, v in out.items() if isinstance(v, float)})
