"""CPU: host halves of the device calibration — Chan's
merge against NumPy's mean / std(ddof=1), the order-key map, and the rank-order
merge of per-rank moments over gloo (world size 2)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_03841_b200 import calib as C


def _moments(x):
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        return C.Moments(0.0, 0.0, 0.0)
    return C.Moments(float(x.size), float(x.mean()), float(((x - x.mean()) ** 2).sum()))


@pytest.mark.parametrize("cuts", [[0, 1000], [0, 1, 2, 1000], [0, 333, 334, 900, 1000], [0, 0, 500, 500, 1000]])
def test_chan_merge_matches_numpy(cuts):
    rng = np.random.default_rng(7)
    x = rng.normal(3e-4, 2e-3, 1000)
    parts = [_moments(x[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    m = C.merge_moments(parts)
    assert m.count == 1000
    assert math.isclose(m.mean, x.mean(), rel_tol=1e-12, abs_tol=1e-18)
    assert math.isclose(m.sigma, x.std(ddof=1), rel_tol=1e-12)


def test_order_key_roundtrip_and_order():
    vals = [-math.inf, -1e300, -2.5, -0.0, 0.0, 1e-310, 3.0, 1e300, math.inf]
    keys = [C._float_to_key(v) for v in vals]
    assert keys == sorted(keys)
    for v, k in zip(vals, keys):
        assert C._key_to_float(k) == v


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, chunks):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = C.RunningStats.__new__(C.RunningStats)
        m = _moments(chunks[rank])
        st.state = torch.tensor([m.count, m.mean, m.m2], dtype=torch.float64)
        q.put((rank, C.merge_stats(st)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_rank_order_merge_world2():
    rng = np.random.default_rng(3)
    x = rng.normal(0.0, 1e-3, 4001)
    chunks = [x[:1700], x[1700:]]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    want = C.merge_moments([_moments(c) for c in chunks])
    for _, m in got:
        assert (m.count, m.mean, m.m2) == (want.count, want.mean, want.m2)
    assert math.isclose(want.sigma, x.std(ddof=1), rel_tol=1e-12)
