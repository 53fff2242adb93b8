import sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT
g = torch.Generator(device='cuda').manual_seed(5)
imgs = torch.randn(256, 3, 224, 224, device='cuda', generator=g)
for dt in (torch.bfloat16, torch.float16, torch.float32):
    m = ProtectedViT(VIT_B16, dtype=dt, seed=1234)
    lg = m(imgs.to(dt)).float()
    top2 = lg.topk(2, dim=1).values
    marg = top2[:, 0] - top2[:, 1]
    pred = lg.argmax(1)
    print(dt, 'distinct classes', pred.unique().numel(), 'logit std over classes', float(lg.std(1).mean()),
          'std over images (per class)', float(lg.std(0).mean()), 'margin mean', float(marg.mean()), 'min', float(marg.min()),
          'nan', bool(lg.isnan().any()))
    h = m.buffers(256).h.float()
    print('   residual stream |h| mean', float(h.abs().mean()), 'max', float(h.abs().max()))
    del m; torch.cuda.empty_cache()
