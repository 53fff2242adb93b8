"""World size 2 on one GPU (two processes, gloo): real campaign shards reduced
through K5 (`distributed.reduce_counters`) equal the single-process campaign —
the reference's toy `run_campaign` (layers split over ranks, merge_campaigns)
and the batched ViT campaign engine (units planned over ranks by suffix cost)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _toy_campaign(rank, world):
    from paper_2310_03841_b200 import distributed as Dd
    from paper_2310_03841_b200 import injector as I
    from paper_2310_03841_b200 import model as Mo
    from paper_2310_03841_b200 import profiler as Pr

    model = Mo.build_toy_model(2, 16, 8, 5, seed=3, dtype="int8")
    ds = Mo.make_synthetic_dataset(model, 12, seed=4)
    golden = Pr.select_golden(model, ds)
    ranges = Pr.profile_ranges(model, ds)
    camp = I.run_campaign(model, golden, ranges, n_per_layer=6, seed=5, rank=rank, world=world)
    t = Dd.counters_tensor({li: {"injections": v[0], "mismatches": v[1]} for li, v in
                            _layer_counts(camp).items()}, len(model.layers), device="cuda")
    return camp, Dd.reduce_counters(t)


def _layer_counts(camp):
    out = {}
    for r in camp.records:
        c = out.setdefault(r.spec.layer_index, [0, 0])
        c[0] += 1
        c[1] += int(r.mismatch)
    return out


def _vit_campaign(rank, world):
    from paper_2310_03841_b200.campaign import ViTCampaign
    from paper_2310_03841_b200.vit import ProtectedViT, ViTConfig

    cfg = ViTConfig(name="mp", dim=256, depth=2, heads=4, mlp=1024, classes=10)
    model = ProtectedViT(cfg, seed=11)
    g = torch.Generator(device="cuda").manual_seed(12)
    cal = [torch.randn(8, 3, 224, 224, device="cuda", generator=g).bfloat16() for _ in range(2)]
    model.calibrate(cal, 1 - 1e-9)
    imgs = torch.randn(8, 3, 224, 224, device="cuda", generator=g).bfloat16()
    camp = ViTCampaign(model, imgs, seed=13, modes=("random_value",))
    return camp.run(2, rank=rank, world_size=world).counters


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        camp, toy_t = _toy_campaign(rank, world)
        vit_c = _vit_campaign(rank, world)
        q.put((rank, camp.to_csv(), toy_t.cpu().tolist(), vit_c.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_world2_campaign_shards_reduce_to_the_single_process_result():
    from paper_2310_03841_b200 import injector as I

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=500) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single_camp, single_toy = _toy_campaign(0, 1)
    single_vit = _vit_campaign(0, 1)
    for rank, csv, toy_t, vit_c in got:
        assert toy_t == single_toy.cpu().tolist()  # K5 over real shards == one process
        assert vit_c == single_vit.tolist()
    merged = I.merge_campaigns([I.CampaignResult.from_csv(c, seed=5, n_per_layer=6) for _, c, _, _ in got])
    assert merged.to_csv() == single_camp.to_csv()
