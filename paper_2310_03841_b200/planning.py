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
Selection follows the reference's rule and summation order (so plans and
their float fields are the reference's bytes): walk the layers by decreasing
vulnerability per unit cost; at every prefix also try completing it with the
cheapest single layer that covers the rest; drop from each candidate the most
expensive picks the target can spare; keep the cheapest candidate.  The
exhaustive search (`method="exact"`, up to 20 candidates) is the optimality
oracle of the tests.

The same module serves the workbench CLI over the reference's toy models
(`cli.py`): `compute_v_orig`, `layer_vulnerabilities`
over a `CampaignResult`, the coverage curves and the checksum / duplication
cost models of a `LayerSpec` (analysis.py:95-133,185-206,297-322).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from itertools import combinations

import numpy as np

__all__ = ["LayerVulnerability", "ProtectionPlan", "CoverageCurve", "layer_macs", "layer_vulnerabilities",
           "checksum_costs", "select_layers", "compute_v_orig", "build_coverage_curve", "checksum_cost_model",
           "duplication_cost_model", "model_totals"]


@dataclass
class LayerVulnerability:
    layer_index: int
    v_orig: float
    p_prop: float
    delta_loss: float
    v_layer: float


_PLAN_FIELDS = ("scheme", "selected", "predicted_coverage", "compute_overhead", "memory_overhead",
                "head_always_included")


@dataclass
class ProtectionPlan:
    """A protected layer set and its predicted coverage / overheads (analysis.py:44-79)."""

    scheme: str
    selected: tuple[int, ...]
    predicted_coverage: float
    compute_overhead: float
    memory_overhead: float
    head_always_included: bool

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in _PLAN_FIELDS}
        d["selected"] = list(self.selected)
        return d

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True)

    @classmethod
    def from_dict(cls, doc: dict) -> "ProtectionPlan":
        kw = {k: doc[k] for k in _PLAN_FIELDS}
        kw["selected"] = tuple(kw["selected"])
        return cls(**kw)

    @classmethod
    def from_json(cls, text: str) -> "ProtectionPlan":
        return cls.from_dict(json.loads(text))


@dataclass
class CoverageCurve:
    """(cumulative overhead, cumulative coverage) as layers are added by value / cost, from (0, 0)."""

    points: list[tuple[float, float]]
    order: list[int]

    def to_csv(self) -> str:
        return "overhead,coverage\n" + "".join(f"{o!r},{c!r}\n" for o, c in self.points)


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


def compute_v_orig(model) -> np.ndarray:
    """MAC share of every layer of a toy `ModelGraph`, summing to 1 (analysis.py:95-98)."""
    from .model import mac_count

    macs = np.array([mac_count(layer) for layer in model.layers], dtype=np.float64)
    return macs / macs.sum()


def _campaign_vulnerabilities(model, campaign) -> list[LayerVulnerability]:
    """analysis.py:101-133 over a `CampaignResult`'s per-layer tallies."""
    share = compute_v_orig(model)
    tallies = campaign.layer_tallies()
    out = []
    for layer in model.layers:
        t = tallies.get(layer.index)
        if not t or t["injections"] == 0:
            raise ValueError(f"no injection records for layer {layer.index}")
        p = t["mismatches"] / t["injections"]
        v = float(share[layer.index])
        out.append(LayerVulnerability(layer.index, v, p, t["loss_delta_sum"] / t["injections"], v * p))
    return out


def layer_vulnerabilities(model, tally) -> list[LayerVulnerability]:
    """V_orig, P_prop, Delta-loss and V_orig * P_prop per layer.

    `tally` is the device campaign's counters (`campaign.Tally`, model a
    `ProtectedViT`) or a host `CampaignResult` (model a toy `ModelGraph`)."""
    if hasattr(tally, "layer_tallies"):
        return _campaign_vulnerabilities(model, tally)
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


def _ratio_order(v: np.ndarray, c: np.ndarray, items) -> list[int]:
    """`items` by decreasing value / cost (zero cost first), then cheaper, then lower index
    (analysis.py:136-140)."""
    with np.errstate(divide="ignore", invalid="ignore"):  # zero costs: the np.where picks inf
        r = np.where(c > 0, v / c, np.inf)
    return sorted(items, key=lambda i: (-r[i], c[i], i))


def _spare(v, c, need: float, picks: list[int]) -> list[int]:
    """Drop the most expensive picks the target can spare (analysis.py:143-151)."""
    kept = list(picks)
    got = sum(float(v[i]) for i in kept)
    for i in sorted(kept, key=lambda j: (-c[j], j)):
        if got - float(v[i]) >= need:
            kept.remove(i)
            got -= float(v[i])
    return kept


def _greedy(v, c, need: float, free: list[int]) -> list[int]:
    """Ratio-ordered prefixes, each also completed by the cheapest single layer covering the
    rest, spared, cheapest kept (analysis.py:154-182)."""
    walk = _ratio_order(v, c, free)
    cands: list[list[int]] = []
    prefix: list[int] = []
    got = 0.0
    for j in range(len(walk) + 1):
        rest = need - got
        if rest <= 0:
            cands.append(list(prefix))
            break
        cover = [i for i in walk[j:] if float(v[i]) >= rest]
        if cover:
            cands.append(prefix + [min(cover, key=lambda i: (c[i], i))])
        if j < len(walk):
            prefix.append(walk[j])
            got += float(v[walk[j]])
    if not cands:
        raise ValueError("coverage target unreachable")
    spared = [_spare(v, c, need, cand) for cand in cands]
    return min(spared, key=lambda s: (sum(float(c[i]) for i in s), len(s), tuple(sorted(s))))


def select_layers(vulns, costs, target_coverage: float, *, head_index: int | None = None, method: str = "greedy",
                  total_compute: float | None = None, memory_costs=None, total_memory: float | None = None,
                  scheme: str = "checksum") -> ProtectionPlan:
    """Cheapest layer set whose vulnerability reaches target_coverage of the total, head forced
    in (analysis.py:213-290; same sums in the same order, so the plan's floats are the reference's)."""
    v = np.asarray(vulns, dtype=np.float64)
    c = np.asarray(costs, dtype=np.float64)
    if not 0.0 < target_coverage <= 1.0:
        raise ValueError("target_coverage must lie in (0, 1]")
    if v.shape != c.shape or v.ndim != 1:
        raise ValueError("vulns and costs must be equal-length vectors")
    total = float(v.sum())
    if total <= 0:
        raise ValueError("total vulnerability is zero")
    forced = set() if head_index is None else {head_index}
    free = [i for i in range(len(v)) if i not in forced]
    if method == "greedy":
        chosen = set(forced)
        got = sum(float(v[i]) for i in forced)
        need = target_coverage * total - got - 1e-12 * total
        if need > 0:
            picks = _greedy(v, c, need, free)
            chosen |= set(picks)
            got += sum(float(v[i]) for i in picks)
        if got / total < target_coverage - 1e-12:
            raise ValueError(f"target coverage {target_coverage} unreachable (max {got / total})")
    elif method == "exact":
        if len(v) > 20:
            raise ValueError("exact selection is limited to 20 layers")
        need = target_coverage * total - sum(float(v[i]) for i in forced)
        best = None
        for r in range(len(free) + 1):
            for combo in combinations(free, r):
                cost, cov = float(sum(c[i] for i in combo)), float(sum(v[i] for i in combo))
                if cov >= need - 1e-12 * total:
                    key = (cost, -cov, combo)
                    best = key if best is None or key < best else best
        if best is None:
            raise ValueError(f"target coverage {target_coverage} unreachable")
        chosen = set(forced) | set(best[2])
        got = sum(float(v[i]) for i in chosen)
    else:
        raise ValueError(f"unknown selection method {method!r}")
    sel = tuple(sorted(chosen))
    cost = float(sum(c[i] for i in sel))
    mem = float(sum(memory_costs[i] for i in sel)) / total_memory if (memory_costs is not None and total_memory) else 0.0
    return ProtectionPlan(scheme, sel, got / total, cost / total_compute if total_compute else cost, mem,
                          head_index is not None)


def build_coverage_curve(vulns, costs, scheme: str = "checksum") -> CoverageCurve:
    """Cumulative coverage against cumulative overhead, layers added by value / cost; coverage
    normalised over the layers given (analysis.py:185-206)."""
    v = np.asarray(vulns, dtype=np.float64)
    c = np.asarray(costs, dtype=np.float64)
    if v.shape != c.shape or v.ndim != 1:
        raise ValueError("vulns and costs must be equal-length vectors")
    if (c < 0).any():
        raise ValueError("costs must be nonnegative")
    total = v.sum()
    order = _ratio_order(v, c, range(len(v)))
    pts = [(0.0, 0.0)]
    oc = ov = 0.0
    for i in order:
        oc += float(c[i])
        ov += float(v[i])
        pts.append((oc, ov / total if total > 0 else 0.0))
    return CoverageCurve(points=pts, order=order)


def checksum_cost_model(layer) -> tuple[float, float]:
    """(flops, memory elements) of checking one toy layer: input and output row sums plus the
    checksum dot product per token; the weight checksum plus two online vectors (analysis.py:297-306)."""
    return float(layer.tokens * (2 * layer.in_dim + layer.out_dim)), float(layer.in_dim + 2 * layer.tokens)


def duplication_cost_model(layer) -> tuple[float, float]:
    """(flops, memory elements) of running one toy layer twice (analysis.py:309-313)."""
    from .model import mac_count

    return (float(2 * mac_count(layer)),
            float(layer.in_dim * layer.out_dim + layer.out_dim + layer.tokens * layer.out_dim))


def model_totals(model) -> tuple[float, float]:
    """(forward flops, resident elements) of a toy model (analysis.py:316-322)."""
    from .model import mac_count

    return (float(sum(2 * mac_count(layer) for layer in model.layers)),
            float(sum(layer.in_dim * layer.out_dim + layer.out_dim + layer.tokens * layer.out_dim
                      for layer in model.layers)))
