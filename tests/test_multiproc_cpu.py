"""CPU, world_size 2 over gloo: the N>1 host logic — sharding covers every unit
exactly once, and the K5 counter all-reduce gives the single-process tallies."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_03841_b200 import distributed as G


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tallies(layers, rank, world):
    """Deterministic per-trial outcomes; each rank counts only its shard of trials."""
    out = {}
    for layer in range(layers):
        mine = G.shard(37 + layer, rank, world)
        t = out.setdefault(layer, {k: 0 for k in G.COUNTER_FIELDS})
        for k in mine:
            t["injections"] += 1
            t["mismatches"] += int((k * 7 + layer) % 5 == 0)
            t["true_positives"] += int((k * 7 + layer) % 5 == 0 and k % 3 != 0)
            t["flagged_rows"] += (k * 13 + layer) % 4
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = G.counters_tensor(_tallies(6, rank, world), 6)
        G.reduce_counters(t)
        q.put((rank, t.tolist(), G.world()))
    finally:
        dist.destroy_process_group()


def test_shard_partitions_units():
    for n in (0, 1, 7, 100):
        for w in (1, 2, 3, 8):
            seen = [u for r in range(w) for u in G.shard(n, r, w)]
            assert seen == list(range(n))


@pytest.mark.timeout(120)
def test_counter_allreduce_world2_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    want = G.counters_tensor(_tallies(6, 0, 1), 6).tolist()
    for rank, t, (r, w) in got:
        assert (r, w) == (rank, 2)
        assert t == want
    assert G.unpack_counters(torch.tensor(want))[0]["injections"] == 37


def test_counters_must_be_int64():
    with pytest.raises(ValueError):
        G.reduce_counters(torch.zeros(3, dtype=torch.float64))
