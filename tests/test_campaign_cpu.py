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


def test_counter_based_draws_are_deterministic_partition_free_and_uniform():
    """The campaign's draws are a function of (seed, layer, k, attempt, draw) only: the same
    value whatever block, shard or vector they are evaluated in; in [0, 1); and uniform."""
    import numpy as np

    from paper_2310_03841_b200.campaign import _uniform

    k = np.arange(4096, dtype=np.uint64)[:, None]
    att = np.arange(4, dtype=np.uint64)[None, :]
    u = _uniform(2310, 7, k, att, 1)
    assert u.shape == (4096, 4) and float(u.min()) >= 0.0 and float(u.max()) < 1.0
    # evaluated alone (another shard / block) -> the same bits
    for kk, aa in ((0, 0), (17, 3), (4095, 2)):
        one = _uniform(2310, 7, np.array([[kk]], dtype=np.uint64), np.array([[aa]], dtype=np.uint64), 1)
        assert one[0, 0] == u[kk, aa]
    # distinct draw index / layer / seed -> different streams
    assert not np.array_equal(u, _uniform(2310, 7, k, att, 2))
    assert not np.array_equal(u, _uniform(2310, 8, k, att, 1))
    assert not np.array_equal(u, _uniform(2311, 7, k, att, 1))
    # uniformity: 16 bins over 16384 draws, chi-square far below the 0.1% critical value (37.7)
    h, _ = np.histogram(u.ravel(), bins=16, range=(0.0, 1.0))
    e = u.size / 16
    assert float(((h - e) ** 2 / e).sum()) < 37.7
