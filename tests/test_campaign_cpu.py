"""Host logic of the batched campaign engine (no GPU): Wilson intervals and
the cost-balanced (layer, block) unit plan shared over ranks."""

from paper_2310_03841_b200.campaign import plan_units, wilson_interval


def test_wilson_and_unit_plan():
    lo, hi = wilson_interval(99, 100)
    assert 0.94 < lo < 0.99 < hi <= 1.0
    units = [(li, b) for li in range(10) for b in range(3)]
    plan = plan_units(units, lambda li: float(10 - li), 4)
    assert sorted(u for p in plan for u in p) == sorted(units)
    loads = [sum(10 - li for li, _ in p) for p in plan]
    assert max(loads) - min(loads) <= 10


def test_unit_plan_is_a_partition_for_every_world_size():
    units = [(li, b) for li in range(50) for b in range(4)]
    for w in (1, 2, 3, 8):
        plan = plan_units(units, lambda li: float(50 - li), w)
        flat = [u for p in plan for u in p]
        assert sorted(flat) == sorted(units) and len(flat) == len(set(flat))
