"""Selective protection planning on host vectors: the plan reaches
its coverage target with the head forced in, greedy never beats the exhaustive oracle, and
the reference's per-layer checksum cost model (analysis.py:297-306) on a ViT-B GEMM list."""

import numpy as np
import pytest

from paper_2310_03841_b200.planning import checksum_costs, layer_macs, select_layers
from paper_2310_03841_b200.vit import VIT_B16


class _M:
    cfg = VIT_B16


def test_select_layers_meets_target_and_forces_head():
    rng = np.random.default_rng(1)
    for trial in range(40):
        n = int(rng.integers(3, 12))
        v = rng.random(n) * (rng.random(n) < 0.8)
        if v.sum() == 0:
            v[0] = 1.0
        c = rng.random(n) + 0.01
        head = n - 1
        for target in (0.3, 0.8, 1.0):
            g = select_layers(v, c, target, head_index=head)
            e = select_layers(v, c, target, head_index=head, method="exact")
            assert head in g.selected and head in e.selected
            assert g.predicted_coverage >= target - 1e-9 and e.predicted_coverage >= target - 1e-9
            assert sum(c[i] for i in e.selected) <= sum(c[i] for i in g.selected) + 1e-12


def test_select_layers_errors():
    with pytest.raises(ValueError, match="target_coverage"):
        select_layers([1.0], [1.0], 0.0)
    with pytest.raises(ValueError, match="zero"):
        select_layers([0.0, 0.0], [1.0, 1.0], 0.5)


def test_vit_b16_cost_model():
    macs = layer_macs(_M())
    comp, mem = checksum_costs(_M())
    assert len(macs) == 50 and abs(2 * macs.sum() - 33.70e9) < 0.01e9  # protected GEMM flops / image
    # checksum work relative to the GEMM: 1/N + 1/(2K) per layer
    assert comp[2] / (2 * macs[2]) == pytest.approx(1 / 768 + 1 / (2 * 768))


def test_planning_matches_reference_golden():
    """select_layers (greedy / exact, cost and memory totals) and build_coverage_curve give the
    reference's bytes on 60 seeded cases (tests/golden/planning.json, written by the reference)."""
    import json
    import warnings
    from pathlib import Path

    from paper_2310_03841_b200.planning import build_coverage_curve

    cases = json.loads((Path(__file__).parent / "golden" / "planning.json").read_text())
    for case in cases:
        v, c, mem = np.array(case["v"]), np.array(case["c"]), np.array(case["mem"])
        for method in ("greedy", "exact"):
            want = case[method]
            if isinstance(want, dict):
                with pytest.raises(ValueError) as exc:
                    select_layers(v, c, case["target"], head_index=case["head"], method=method,
                                  total_compute=case["total_compute"], memory_costs=mem,
                                  total_memory=case["total_memory"])
                assert str(exc.value) == want["error"]
            else:
                got = select_layers(v, c, case["target"], head_index=case["head"], method=method,
                                    total_compute=case["total_compute"], memory_costs=mem,
                                    total_memory=case["total_memory"])
                assert got.to_json() == want
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)  # 0 / 0 ratios, as in the reference
            assert build_coverage_curve(v, c).to_csv() == case["curve"]
