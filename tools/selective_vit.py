"""Vulnerability ranking and selective protection on ViT-B/16 b256:
a random-value output-fault campaign (device counters) -> per-layer V_orig, P_prop, Delta-loss
-> protection plans for several coverage targets (head forced) -> each plan applied
(ProtectedViT.set_protected): protected-forward overhead against the unprotected forward and the
realised coverage of a fresh validation campaign (mismatches from unprotected layers count as missed)."""
import json, statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200.campaign import ViTCampaign, select_golden_images, wilson_interval
from paper_2310_03841_b200.planning import checksum_costs, layer_macs, layer_vulnerabilities, select_layers
from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT

B, blocks = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device('cuda')
g = torch.Generator(device=dev).manual_seed(11)
img = lambda: torch.randn(B, 3, 224, 224, device=dev, generator=g).bfloat16()  # noqa: E731
m = ProtectedViT(VIT_B16, seed=1234)
m.calibrate([img(), img()], 1 - 1e-9)
teacher = ProtectedViT(VIT_B16, dtype=torch.float32, seed=1234)
golden, gstats = select_golden_images(m, teacher, img, B)
del teacher; torch.cuda.empty_cache()
modes = ("random_value",)
tally = ViTCampaign(m, golden, seed=1, modes=modes).run(blocks)
vul = layer_vulnerabilities(m, tally)
macs = layer_macs(m); comp, mem = checksum_costs(m)
head = VIT_B16.n_layers - 1


def timed(gr, n=10):
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def graph(protect):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): m(golden, protect=protect)
    torch.cuda.synchronize(); gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s): m(golden, protect=protect)
    return gr


out = {"golden": gstats, "campaign": tally.summary(), "modes": modes,
       "vulnerability": [{"layer": v.layer_index, "v_orig": v.v_orig, "p_prop": v.p_prop, "delta_loss": v.delta_loss,
                          "v_layer": v.v_layer} for v in vul], "plans": []}
gu = graph(False)
for target in (0.5, 0.9, 0.99, 1.0):
    plan = select_layers([v.v_layer for v in vul], comp, target, head_index=head, total_compute=2 * macs.sum(),
                         memory_costs=mem)
    m.set_protected(plan.selected)
    gp = graph(True)
    tp_, tu_ = [], []
    for r in range(6):
        for gr, acc in (((gp, tp_), (gu, tu_)) if r % 2 == 0 else ((gu, tu_), (gp, tp_))):
            acc.append(timed(gr))
    ov = 100 * (statistics.median(tp_) / statistics.median(tu_) - 1)
    val = ViTCampaign(m, golden, seed=2, modes=modes).run(max(1, blocks // 2))
    tp, fn = val.total("true_positives"), val.total("false_negatives")
    out["plans"].append({"target": target, "layers": len(plan.selected), "selected": list(plan.selected),
                         "predicted_coverage": plan.predicted_coverage,
                         "checksum_flops_share": plan.compute_overhead, "measured_overhead_pct": ov,
                         "validation_mismatches": tp + fn, "validation_coverage": tp / (tp + fn) if tp + fn else 1.0,
                         "validation_wilson95": wilson_interval(tp, tp + fn)})
    del gp
m.set_protected(range(VIT_B16.n_layers))
print(json.dumps(out))
