"""GPU: gg_running_stats and gg_minmax against NumPy /
torch on the same inputs."""

import math

import numpy as np
import pytest
import torch

from paper_2310_03841_b200 import calib as C

pytestmark = pytest.mark.gpu


def test_running_stats_matches_numpy_over_batches_and_is_deterministic():
    g = torch.Generator(device="cpu").manual_seed(0)
    batches = [torch.randn(n, generator=g, dtype=torch.float64) * 1e-3 + 2e-4 for n in (1, 50432, 7, 3000, 1025)]
    states = []
    for _ in range(2):
        st = C.RunningStats("cuda")
        for b in batches:
            st.update(b.cuda())
        states.append(st.state.cpu())
    assert torch.equal(states[0].view(torch.int64), states[1].view(torch.int64))
    allx = torch.cat(batches).numpy()
    m = C.RunningStats.moments(type("S", (), {"state": states[0]})())
    assert m.count == allx.size
    assert math.isclose(m.mean, allx.mean(), rel_tol=1e-12)
    assert math.isclose(m.sigma, allx.std(ddof=1), rel_tol=1e-11)
    st = C.RunningStats("cuda")
    for b in batches:
        st.update(b.cuda())
    mu, lo, hi = st.epsilon(0.9999)
    assert lo < mu < hi


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int32])
@pytest.mark.parametrize("shape,pitch", [((50432, 768), 768), ((197, 3072), 3072), ((33, 101), 101), ((40, 96), 128)])
def test_minmax_matches_torch(dtype, shape, pitch):
    M, N = shape
    g = torch.Generator(device="cpu").manual_seed(M + N)
    if dtype == torch.int32:
        base = torch.randint(-2**30, 2**30, (M, pitch), generator=g, dtype=torch.int32)
    else:
        base = (torch.randn(M, pitch, generator=g) * 7).to(dtype)
    y = base.cuda()[:, :N]
    rr = C.RunningRange("cuda")
    rr.update(y)
    lo, hi, bad = rr.bounds()
    ref = y.double()
    assert lo == ref.min().item() and hi == ref.max().item() and bad == 0


def test_minmax_counts_non_finite_and_accumulates():
    y = torch.randn(64, 64, device="cuda", dtype=torch.float32)
    y[3, 5] = float("nan")
    y[7, 9] = float("inf")
    y[1, 1] = -float("inf")
    rr = C.RunningRange("cuda")
    rr.update(y)
    y2 = torch.full((8, 16), 100.0, device="cuda")
    rr.update(y2)
    lo, hi, bad = rr.bounds()
    finite = y[torch.isfinite(y)].double()
    assert bad == 3 and lo == finite.min().item() and hi == 100.0
