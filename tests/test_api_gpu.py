"""GPU: the reference's conformance tests for the hot path (category A of
SURVEY.md §4 — order-independent behaviour), restated against the B200
package: integer soundness, replay exactness, clean-path identity, skip
policies, error messages, sampler rules, campaign determinism and the
statistical false-positive bound.  Tensor engine (default) throughout."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2310_03841_b200 import guard as G  # noqa: E402
from paper_2310_03841_b200.errors import GuardError, SamplingError  # noqa: E402
from paper_2310_03841_b200.guard import (  # noqa: E402
    CorrectionPolicy,
    EpsilonModel,
    calibrate_epsilon,
    detection_guarantee,
    evaluate_detection,
    offline_checksum,
    protected_forward,
    verify_layer,
)
from paper_2310_03841_b200.injector import (  # noqa: E402
    CampaignResult,
    InjectionSpec,
    inject_forward,
    injected_forward,
    merge_campaigns,
    run_campaign,
    sample_injection,
)
from paper_2310_03841_b200.model import (  # noqa: E402
    LayerSpec,
    build_toy_model,
    forward,
    make_synthetic_dataset,
)
from paper_2310_03841_b200.numerics import Matrix2D, Precision, flip_bit, gemm, reduce_cols, reduce_rows  # noqa: E402
from paper_2310_03841_b200.profiler import RangeProfile, profile_ranges, select_golden  # noqa: E402


def _layer(wt, bias, dtype="binary64", tokens=2):
    w = Matrix2D(wt, dtype)
    return LayerSpec(0, "L0", "embed", w.rows, w.cols, tokens, w, np.asarray(bias))


@pytest.fixture(scope="module")
def fp16_bench():
    model = build_toy_model(blocks=1, dim=8, tokens=4, classes=5, seed=41, dtype="binary16-emulated")
    ds = make_synthetic_dataset(model, 40, seed=4)
    golden = select_golden(model, ds)
    ranges = profile_ranges(model, ds)
    chks = {L.index: offline_checksum(L, Precision.BINARY64) for L in model.layers}
    eps = calibrate_epsilon(model, golden, confidence=0.9999)
    return model, golden, ranges, chks, eps


@pytest.fixture(scope="module")
def fp32_bench():
    model = build_toy_model(blocks=1, dim=8, tokens=4, classes=5, seed=29)
    ds = make_synthetic_dataset(model, 12, seed=2)
    return model, select_golden(model, ds), profile_ranges(model, ds)


# ------------------------------------------------------------- numerics
def test_gemm_known_answers_all_engines():
    for engine in ("tensor", "exact"):
        assert gemm(Matrix2D([[1, 2], [3, 4]], "int8"), Matrix2D([[5, 6], [7, 8]], "int8"),
                    engine=engine).tolist() == [[19, 22], [43, 50]]
    assert gemm(Matrix2D([[1, 2], [3, 4]]), Matrix2D([[5, 6], [7, 8]]), accum=Precision.BINARY64).tolist() == \
        [[19, 22], [43, 50]]
    assert gemm(Matrix2D([[1, 1]]), Matrix2D([[1, 2], [3, 4]]), bias=[1, 1],
                accum=Precision.BINARY64).tolist() == [[5, 7]]
    x16 = Matrix2D([[1.0, 2.0]], "binary16-emulated")
    assert gemm(x16, Matrix2D([[0.5], [0.25]], "binary16-emulated")).tolist() == [[1.0]]


def test_gemm_errors_match_reference_messages():
    with pytest.raises(ValueError, match="dims"):
        gemm(Matrix2D([[1, 2]]), Matrix2D([[1, 2]]))
    with pytest.raises(ValueError, match="bias"):
        gemm(Matrix2D([[1, 2]]), Matrix2D([[1], [2]]), bias=[1, 2])
    with pytest.raises(ValueError, match="narrower"):
        gemm(Matrix2D([[1.0]]), Matrix2D([[1.0]]), accum=Precision.BINARY32)
    h = Matrix2D([[1.0]], "binary16-emulated")
    with pytest.raises(ValueError, match="binary32 or wider"):
        gemm(h, h, accum=Precision.BINARY16)
    with pytest.raises(ValueError, match="int64-exact"):
        gemm(Matrix2D([[1]], "int8"), Matrix2D([[1]], "int8"), accum=Precision.BINARY64)


def test_gemm_deterministic_tensor_engine():
    rng = np.random.default_rng(7)
    X = Matrix2D(rng.standard_normal((300, 96)).astype(np.float32), "binary32")
    W = Matrix2D(rng.standard_normal((96, 520)).astype(np.float32), "binary32")
    assert gemm(X, W) == gemm(X, W)


def test_reductions_match_ascending_folds():
    assert reduce_rows(Matrix2D([[1, 2], [3, 4]])).tolist() == [3, 7]
    assert reduce_cols(Matrix2D([[1, 2], [3, 4]])).tolist() == [4, 6]
    rng = np.random.default_rng(99)
    M = Matrix2D(rng.standard_normal((8, 8)).astype(np.float32), "binary32")
    r = reduce_rows(M)
    for b in range(8):
        acc = 0.0
        for v in M.data[b]:
            acc += float(v)
        assert r[b] == acc
    Mi = Matrix2D(rng.integers(-(2**20), 2**20, (6, 9)), "int32")
    assert int(reduce_rows(Mi).sum()) == int(reduce_cols(Mi).sum())


# ------------------------------------------------------- checksum / verify
def test_integer_checksum_algebra_exact():
    rng = np.random.default_rng(8)
    for _ in range(40):
        X = Matrix2D(rng.integers(-100, 101, (3, 9)), "int8")
        L = _layer(rng.integers(-100, 101, (9, 5)), rng.integers(-50, 51, 5), "int8", 3)
        Y = gemm(X, L.weight, bias=L.bias, accum=Precision.INT64)
        out = verify_layer(X, Y, offline_checksum(L, Precision.INT64))
        assert np.all(out.d == 0) and not out.triggered


def test_integer_flip_detection_is_exhaustive():
    """Every value-changing flip of Y, X or a weight scratch copy trips the exact check."""
    rng = np.random.default_rng(15)
    X = Matrix2D(rng.integers(-100, 101, (2, 4)), "int8")
    L = _layer(rng.integers(-100, 101, (4, 3)), rng.integers(-5, 6, 3), "int8", 2)
    chk = offline_checksum(L, Precision.INT64)
    assert np.all(chk.w_sum != 0)
    Y = gemm(X, L.weight, bias=L.bias, accum=Precision.INT64)
    for e in range(Y.data.size):
        for bit in range(32):
            yc = Y.copy()
            yc.data.reshape(-1)[e] = flip_bit(yc.data.reshape(-1)[e], bit, "int32")
            assert verify_layer(X, yc, chk).triggered
    for e in range(X.data.size):
        for bit in range(8):
            xc = X.copy()
            xc.data.reshape(-1)[e] = flip_bit(xc.data.reshape(-1)[e], bit, "int8")
            assert verify_layer(xc, Y, chk).triggered
    for e in range(L.weight.data.size):
        wc = L.weight.copy()
        wc.data.reshape(-1)[e] = flip_bit(wc.data.reshape(-1)[e], 3, "int8")
        yc = gemm(X, wc, bias=L.bias, accum=Precision.INT64)
        assert verify_layer(X, yc, chk).triggered == bool(np.any(X.data[:, e // L.out_dim] != 0))
    assert not verify_layer(X, Y, chk).triggered


def test_verify_argument_errors():
    L = _layer([[1.0]], [0.0])
    chk = offline_checksum(L, Precision.BINARY64)
    with pytest.raises(ValueError, match="epsilon"):
        verify_layer(Matrix2D([[1.0]]), Matrix2D([[1.0]]), chk)
    L2 = _layer([[1.0, 2.0]], [0.0, 0.0])
    eps = EpsilonModel(0, 0.0, 1.0, 0.95, -2.0, 2.0, 100, Precision.BINARY64)
    with pytest.raises(ValueError, match="cols"):
        verify_layer(Matrix2D([[1.0, 2.0]]), Matrix2D([[1.0, 2.0]]), offline_checksum(L2, Precision.BINARY64), eps)
    with pytest.raises(ValueError, match="int64-exact"):
        offline_checksum(_layer([[1, 2]], [0, 0], "int8"), Precision.BINARY64)


# ----------------------------------------------------------- calibration
def test_calibrate_int_model_degenerates_to_exact():
    model = build_toy_model(blocks=1, dim=8, tokens=4, classes=4, seed=6, dtype="int8")
    golden = select_golden(model, make_synthetic_dataset(model, 5, seed=2))
    for m in calibrate_epsilon(model, golden).values():
        assert m.precision is Precision.INT64 and (m.mu, m.sigma, m.threshold_low, m.threshold_high) == (0, 0, 0, 0)


def test_calibrate_matches_brute_force(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    layer, got = 2, []
    for sid in golden.sample_ids:
        t = forward(model, golden.input_for(sid), golden.labels[sid], tap=[layer])
        x, y, w = t.inputs[layer].widened(), t.outputs[layer].widened(), chks[layer].w_sum
        for b in range(x.shape[0]):
            pred = 0.0
            for k in range(x.shape[1]):
                pred += x[b, k] * w[k]
            pred += chks[layer].bias_sum
            obs = 0.0
            for o in range(y.shape[1]):
                obs += y[b, o]
            got.append(pred - obs)
    got = np.array(got)
    assert eps[layer].mu == pytest.approx(got.mean(), rel=1e-12, abs=1e-15)
    assert eps[layer].sigma == pytest.approx(got.std(ddof=1), rel=1e-12)
    assert eps[layer].n_samples == len(got)


def test_calibrate_requires_30_samples():
    from paper_2310_03841_b200.errors import CalibrationError

    model = build_toy_model(blocks=1, dim=8, tokens=4, classes=4, seed=7, dtype="binary16-emulated")
    golden = select_golden(model, make_synthetic_dataset(model, 3, seed=3))
    with pytest.raises(CalibrationError, match="< 30"):
        calibrate_epsilon(model, golden, per_sample=False)


# ------------------------------------------------------ protected forward
def test_clean_path_identity(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    every = list(range(len(model.layers)))
    for sid in golden.sample_ids[:10]:
        x, label = golden.input_for(sid), golden.labels[sid]
        plain = forward(model, x, label)
        guarded, events = protected_forward(model, x, label, every, chks, eps, CorrectionPolicy("replay"))
        assert guarded.logits.tobytes() == plain.logits.tobytes() and guarded.loss == plain.loss


def test_detect_and_replay_restores_clean_logits(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    sid = golden.sample_ids[0]
    x, label = golden.input_for(sid), golden.labels[sid]
    target = float(forward(model, x, label, tap=[2]).outputs[2].widened().ravel()[3])
    spec = InjectionSpec(2, "output", 3, None, "fixed_value", sid, 0, value=target + 1024.0)
    guarded, events = protected_forward(model, x, label, list(range(len(model.layers))), chks, eps,
                                        CorrectionPolicy("replay", max_replays=3), inject=spec)
    assert [(e.layer_index, e.action) for e in events if e.triggered] == [(2, "replay")]
    assert guarded.logits.tobytes() == forward(model, x, label).logits.tobytes()


def test_bit_flip_output_fault_in_epilogue_is_detected(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    sid = golden.sample_ids[1]
    x, label = golden.input_for(sid), golden.labels[sid]
    spec = InjectionSpec(3, "output", 5, 14, "fp_exponent_bit", sid, 0)  # top exponent bit of fp16
    _, events = protected_forward(model, x, label, list(range(len(model.layers))), chks, eps, None, inject=spec)
    ev = [e for e in events if e.layer_index == 3]
    assert ev and ev[0].action == "detect" and ev[0].flagged_rows == 1


def test_numerical_false_alarm_is_accepted(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    tight = {i: EpsilonModel(i, m.mu, 0.0, m.confidence, m.mu, m.mu, m.n_samples, m.precision)
             for i, m in eps.items()}
    sid = golden.sample_ids[2]
    x, label = golden.input_for(sid), golden.labels[sid]
    guarded, events = protected_forward(model, x, label, list(range(len(model.layers))), chks, tight,
                                        CorrectionPolicy("replay", max_replays=2))
    assert any(e.action == "replay_numerical" for e in events)
    assert guarded.logits.tobytes() == forward(model, x, label).logits.tobytes()


def test_replay_budget_exhaustion(fp16_bench, monkeypatch):
    model, golden, _, chks, eps = fp16_bench
    real = G.run_layer
    n = {"calls": 0}

    def flaky(m, layer, xin):
        y = real(m, layer, xin)
        if layer.index == 2:
            n["calls"] += 1
            y = y.copy()
            y.reshape(-1)[0] += 100.0 * n["calls"]
        return y

    monkeypatch.setattr(G, "run_layer", flaky)
    sid = golden.sample_ids[0]
    with pytest.raises(GuardError, match="replay budget"):
        protected_forward(model, golden.input_for(sid), golden.labels[sid], [2], chks, eps,
                          CorrectionPolicy("replay", max_replays=2))


def test_skip_policies(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    sid = golden.sample_ids[0]
    x, label = golden.input_for(sid), golden.labels[sid]
    every = list(range(len(model.layers)))
    t1 = float(forward(model, x, label, tap=[1]).outputs[1].widened().ravel()[0])
    spec = InjectionSpec(1, "output", 0, None, "fixed_value", sid, 0, value=t1 + 1000.0)
    _, events = protected_forward(model, x, label, every, chks, eps, CorrectionPolicy("skip_same_size"), inject=spec)
    skips = [e for e in events if e.action == "skip"]
    assert len(skips) == 1 and skips[0].skip_target == 2
    fc2 = next(L.index for L in model.layers if L.kind == "mlp_fc2")
    t2 = float(forward(model, x, label, tap=[fc2]).outputs[fc2].widened().ravel()[0])
    spec2 = InjectionSpec(fc2, "output", 0, None, "fixed_value", sid, 0, value=t2 + 1000.0)
    with pytest.raises(GuardError, match="does not fit the head"):
        protected_forward(model, x, label, [fc2], chks, eps, CorrectionPolicy("skip_to_head"), inject=spec2)
    with pytest.raises(ValueError, match="lacks"):
        protected_forward(model, x, label, [0], {}, eps, None)


def test_unprotected_layer_forfeits_coverage(fp16_bench):
    model, golden, _, chks, eps = fp16_bench
    sid = golden.sample_ids[1]
    x, label = golden.input_for(sid), golden.labels[sid]
    t = float(forward(model, x, label, tap=[3]).outputs[3].widened().ravel()[0])
    spec = InjectionSpec(3, "output", 0, None, "fixed_value", sid, 0, value=t + 500.0)
    protected = [i for i in range(len(model.layers)) if i != 3]
    _, events = protected_forward(model, x, label, protected, chks, eps, CorrectionPolicy("replay"), inject=spec)
    assert all(e.layer_index != 3 for e in events)


# -------------------------------------------------------------- campaigns
def test_evaluate_detection_tallies_and_guarantee(fp16_bench):
    model, golden, ranges, chks, eps = fp16_bench
    rep = evaluate_detection(model, golden, range(len(model.layers)), chks, eps, ranges, n_per_layer=30, seed=11,
                             clean_passes=5)
    assert rep.true_positives + rep.false_negatives + rep.benign_detections + rep.true_negatives == len(rep.records)
    checked = 0
    for r in rep.records:
        if abs(r.corrupted_value - r.original_value) > detection_guarantee(eps[r.spec.layer_index],
                                                                           model.layers[r.spec.layer_index], ranges):
            checked += 1
            assert r.detected
    assert checked > 0
    assert rep.to_csv().count("\n") == len(rep.records) + 1


def test_evaluate_detection_huge_faults_all_detected(fp16_bench):
    model, golden, ranges, chks, eps = fp16_bench
    wide = RangeProfile({i: (lo - 1e4, hi + 1e4) for i, (lo, hi) in ranges.bounds.items()})
    rep = evaluate_detection(model, golden, range(len(model.layers)), chks, eps, wide, n_per_layer=5,
                             modes=("random_value",), seed=3, clean_passes=5)
    big = [r for r in rep.records if abs(r.corrupted_value - r.original_value) > 1e3]
    assert big and all(r.detected for r in big)


def test_false_positive_rate_bound(fp16_bench):
    model, _, _, chks, _ = fp16_bench
    eps = calibrate_epsilon(model, select_golden(model, make_synthetic_dataset(model, 60, seed=100)),
                            confidence=0.99)
    held = select_golden(model, make_synthetic_dataset(model, 60, seed=200))
    flags = checks = 0
    for sid in held.sample_ids:
        _, events = protected_forward(model, held.input_for(sid), held.labels[sid], list(range(len(model.layers))),
                                      chks, eps, None, record_all=True)
        for ev in events:
            checks += model.layers[ev.layer_index].tokens
            flags += ev.flagged_rows
    assert flags / checks <= 0.01 + 3.0 * math.sqrt(0.01 * 0.99 / checks)


def test_sampler_rules(fp32_bench):
    model, golden, ranges = fp32_bench
    rng = np.random.default_rng(1)
    for _ in range(150):
        layer = int(rng.integers(len(model.layers)))
        spec = sample_injection(model, ranges, golden, rng, layer_index=layer)
        rec = inject_forward(model, golden.input_for(spec.sample_id), golden.labels[spec.sample_id], spec)
        lo, hi = ranges.bounds[layer]
        assert lo <= rec.corrupted_value <= hi and rec.corrupted_value != rec.original_value
    with pytest.raises(SamplingError, match="layer 0"):
        sample_injection(model, RangeProfile({i: (0.0, 0.0) for i in range(len(model.layers))}), golden,
                         np.random.default_rng(3), layer_index=0)


def test_injection_locality_and_transience(fp32_bench):
    model, golden, ranges = fp32_bench
    sid = golden.sample_ids[0]
    x, label = golden.input_for(sid), golden.labels[sid]
    every = tuple(range(len(model.layers)))
    clean = forward(model, x, label, tap=every)
    spec = sample_injection(model, ranges, golden, np.random.default_rng(11), layer_index=3, sample_id=sid)
    trace, _, _ = injected_forward(model, x, label, spec, tap=every)
    for i in range(3):
        assert trace.outputs[i] == clean.outputs[i] and trace.inputs[i] == clean.inputs[i]
    before = model.layers[1].weight.data.tobytes()
    inject_forward(model, x, label, InjectionSpec(1, "weight", 9, 20, "fp_exponent_bit", sid, 0))
    assert model.layers[1].weight.data.tobytes() == before
    t, orig, bad = injected_forward(model, x, label, InjectionSpec(2, "input", 4, None, "fixed_value", sid, 0,
                                                                   value=3.75), tap=(2,))
    assert bad == 3.75 and t.inputs[2].widened().ravel()[4] == 3.75


def test_campaign_determinism_sharding_and_csv(fp32_bench):
    model, golden, ranges = fp32_bench
    a = run_campaign(model, golden, ranges, 5, seed=77)
    assert a.to_csv() == run_campaign(model, golden, ranges, 5, seed=77).to_csv()
    shards = [run_campaign(model, golden, ranges, 5, seed=77, rank=r, world=3) for r in range(3)]
    assert merge_campaigns(shards).to_csv() == a.to_csv()
    back = CampaignResult.from_csv(a.to_csv(), seed=77, n_per_layer=5)
    assert back.to_csv() == a.to_csv()
    t = a.layer_tallies()
    for layer in range(len(model.layers)):
        assert t[layer]["injections"] + a.skipped.get(layer, 0) == 5


def test_int8_campaign(fp32_bench):
    model = build_toy_model(blocks=1, dim=8, tokens=4, classes=4, seed=3, dtype="int8")
    ds = make_synthetic_dataset(model, 8, seed=1)
    golden, ranges = select_golden(model, ds), profile_ranges(model, ds)
    for rec in run_campaign(model, golden, ranges, 10, seed=9).records:
        lo, hi = ranges.bounds[rec.spec.layer_index]
        assert isinstance(rec.original_value, int) and lo <= rec.corrupted_value <= hi


def test_fused_check_takes_the_chosen_checksum_precisions(fp16_bench):
    """choose_checksum_precision's binary32 / binary16 picks run the fused check (no extra verify
    pass); its d stays within the reference-precision fold's error of the reference d, and a fault
    is still detected."""
    from paper_2310_03841_b200 import guard as GG
    from paper_2310_03841_b200.model import CheckedOutput

    model, golden, ranges, _, _ = fp16_bench
    for p in (Precision.BINARY32, Precision.BINARY16):
        chks = {L.index: offline_checksum(L, p) for L in model.layers}
        eps = calibrate_epsilon(model, golden, precisions=p, confidence=0.9999)
        sid = golden.sample_ids[0]
        x, label = golden.input_for(sid), golden.labels[sid]
        seen = []
        real = GG._verify_arrays

        def spy(xin, y, chk, e):
            seen.append(isinstance(y, CheckedOutput) and y.fused_verdict() is not None)
            return real(xin, y, chk, e)

        GG._verify_arrays = spy
        try:
            _, events = protected_forward(model, x, label, list(range(len(model.layers))), chks, eps, None,
                                          record_all=True)
        finally:
            GG._verify_arrays = real
        assert seen and all(seen)  # every check came from the fused launch
        spec = InjectionSpec(2, "output", 3, 14, "fp_exponent_bit", sid, 0)
        _, events = protected_forward(model, x, label, list(range(len(model.layers))), chks, eps, None, inject=spec)
        assert [e.layer_index for e in events if e.triggered] == [2]


@pytest.mark.parametrize("name", ["toy_fp16.albt", "toy_int8.albt", "toy_fp32.albt"])
def test_albt_loads_into_device_memory(name):
    """One host->device transfer of the reference-written container; device weights in K1's
    [out, in] layout equal the host model's; K2 on the device gives the reference checksums."""
    import torch

    from paper_2310_03841_b200 import albt
    from tests.golden_io import GOLDEN

    model = albt.load_model(GOLDEN / name)
    dw = albt.load_device(GOLDEN / name)
    for ly in model.layers:
        w = dw.weights[ly.index].cpu().numpy()
        assert np.array_equal(w.T.astype(np.float64), ly.weight.widened())
        p = Precision.INT64 if model.is_integer else Precision.BINARY64
        chk = offline_checksum(ly, p)
        assert dw.w_sum[ly.index].cpu().numpy().tobytes() == chk.w_sum.tobytes()
        assert dw.bias_sum[ly.index] == chk.bias_sum

