"""Layer vulnerability ranking and selective protection over the device
campaign counters.

The quantities are the reference's (/root/reference/pkg/src/gemmguard/
analysis.py): a layer's origination share V_orig is its fraction of the
model's multiply-accumulates (analysis.py:95-98), its propagation rate P_prop
the fraction of its injections that changed the predicted class
(analysis.py:101-106), Delta-loss the mean loss shift (analysis.py:109-114) and
its vulnerability V_orig * P_prop (analysis.py:117-133).  A protection plan is
a layer set whose summed vulnerability reaches a target share of the total at
the lowest checksum cost, the classifier head always included (PAPER.md:473,
analysis.py:213-290); the per-layer checksum cost is the reference's model
(input and output row reductions plus the checksum dot product per token,
analysis.py:297-306).

Here the counters come from the batched device campaign (`campaign.py`,
all-reduced across ranks by K5), the model is a `ProtectedViT` (its GEMM list
gives the MAC counts) and a plan is applied with `ProtectedViT.set_protected`.
Selection: layers by decreasing vulnerability per unit cost until the target
is met, then the most expensive picks the target can spare are dropped; the
exhaustive search (`method="exact"`, up to 20 candidates) is the optimality
oracle of the tests.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass
from itertools import combinations

import numpy as np

__all__ = ["LayerVulnerability", "ProtectionPlan", "layer_macs", "layer_vulnerabilities", "checksum_costs",
           "select_layers"]


@dataclass
class LayerVulnerability:
    layer_index: int
    v_orig: float
    p_prop: float
    delta_loss: float
    v_layer: float


@dataclass
class ProtectionPlan:
    scheme: str
    selected: tuple[int, ...]
    predicted_coverage: float
    compute_overhead: float
    memory_overhead: float
    head_always_included: bool

    def to_json(self) -> str:
        d = asdict(self)
        d["selected"] = list(self.selected)
        return json.dumps(d, indent=2, sort_keys=True)


def layer_macs(model) -> np.ndarray:
    """Multiply-accumulates of every protected layer for one image (the model's GEMM list)."""
    return np.array([float(M) * N * K for _, M, N, K, *_ in model.cfg.gemms(1)], dtype=np.float64)


def checksum_costs(model) -> tuple[np.ndarray, np.ndarray]:
    """Per layer and image: checksum flops tokens * (2 in + out) and memory in + 2 tokens."""
    comp, mem = [], []
    for _, M, N, K, *_ in model.cfg.gemms(1):
        comp.append(float(M) * (2 * K + N))
        mem.append(float(K) + 2.0 * M)
    return np.array(comp), np.array(mem)


def layer_vulnerabilities(model, tally) -> list[LayerVulnerability]:
    """V_orig, P_prop, Delta-loss and V_orig * P_prop per layer from a campaign's counters."""
    macs = layer_macs(model)
    share = macs / macs.sum()
    out = []
    for i in range(len(macs)):
        t = tally.layer(i)
        if t["injections"] == 0:
            raise ValueError(f"no injection records for layer {i}")
        p = t["mismatches"] / t["injections"]
        out.append(LayerVulnerability(i, float(share[i]), p, t["delta_loss"], float(share[i]) * p))
    return out


def select_layers(vulns, costs, target_coverage: float, *, head_index: int | None = None, method: str = "greedy",
                  total_compute: float | None = None, memory_costs=None, total_memory: float | None = None,
                  scheme: str = "checksum") -> ProtectionPlan:
    """Cheapest layer set whose vulnerability reaches target_coverage of the total (head forced in)."""
    v = np.asarray(vulns, dtype=np.float64)
    c = np.asarray(costs, dtype=np.float64)
    if not 0.0 < target_coverage <= 1.0:
        raise ValueError("target_coverage must lie in (0, 1]")
    if v.shape != c.shape or v.ndim != 1:
        raise ValueError("vulns and costs must be equal-length vectors")
    total = float(v.sum())
    if total <= 0:
        raise ValueError("total vulnerability is zero")
    forced = [] if head_index is None else [head_index]
    need = target_coverage * total * (1.0 - 1e-12)
    free = [i for i in range(len(v)) if i not in forced]
    base = float(sum(v[i] for i in forced))
    if method == "greedy":
        ratio = {i: (v[i] / c[i] if c[i] > 0 else np.inf) for i in free}
        chosen, got = [], base
        for i in sorted(free, key=lambda j: (-ratio[j], c[j], j)):
            if got >= need:
                break
            chosen.append(i)
            got += float(v[i])
        if got < need:
            raise ValueError(f"target coverage {target_coverage} unreachable")
        for i in sorted(chosen, key=lambda j: (-c[j], j)):  # drop what the target can spare
            if got - float(v[i]) >= need:
                chosen.remove(i)
                got -= float(v[i])
        picked = chosen
    elif method == "exact":
        if len(v) > 20:
            raise ValueError("exact selection is limited to 20 layers")
        best = None
        for r in range(len(free) + 1):
            for combo in combinations(free, r):
                cov = base + float(sum(v[i] for i in combo))
                if cov >= need:
                    key = (float(sum(c[i] for i in combo)), -cov, combo)
                    best = key if best is None or key < best else best
        if best is None:
            raise ValueError(f"target coverage {target_coverage} unreachable")
        picked = list(best[2])
    else:
        raise ValueError(f"unknown selection method {method!r}")
    sel = tuple(sorted(set(forced) | set(picked)))
    cost = float(sum(c[i] for i in sel))
    mem = float(sum(memory_costs[i] for i in sel)) / total_memory if (memory_costs is not None and total_memory) else 0.0
    return ProtectionPlan(scheme, sel, float(sum(v[i] for i in sel)) / total,
                          cost / total_compute if total_compute else cost, mem, head_index is not None)
