"""GPU parity: the B200 path against the reference's own outputs (golden
fixtures made by running the reference, tests/golden/make_golden.py) and the
oracle, on identical seeded inputs.

Bars: bit-exact for int8 / integer work, for the offline checksum, for the
reference-order verification, for flips and for everything computed by the
"exact" engine; floating-point tensor-core GEMMs within the fp32-accumulation
bound stated in `_fp_tolerance` (fp16/bf16 operands are exact in fp32, so the
only error is the accumulation order: |dy| <= K * 2^-23 * sum|x w| + 1 ulp of
the output; binary32 operands run as 3xTF32 and add <= 2^-20 * sum|x w|)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import gemmguard_oracle as O  # noqa: E402
from paper_2310_03841_b200 import guard as G  # noqa: E402
from paper_2310_03841_b200 import injector as I  # noqa: E402
from paper_2310_03841_b200 import model as Mo  # noqa: E402
from paper_2310_03841_b200 import profiler as Pr  # noqa: E402
from paper_2310_03841_b200.numerics import Matrix2D, Precision, gemm  # noqa: E402
from tests.golden_io import cfg1_inputs, doc, gemm_case_inputs, npz, sha  # noqa: E402


@pytest.fixture
def exact_engine(monkeypatch):
    monkeypatch.setenv("GEMMGUARD_ENGINE", "exact")


def _fp_tolerance(x, wt, bias, y_ref, dtype):
    mag = np.abs(x.astype(np.float64)) @ np.abs(wt.astype(np.float64)) + np.abs(bias)
    K = x.shape[1]
    ulp = {"binary16-emulated": 2.0**-10, "binary32": 2.0**-23}[dtype]
    tf32 = 2.0**-20 if dtype == "binary32" else 0.0  # 3xTF32: lo*lo dropped, lo tf32-truncated
    return mag * (K * 2.0**-23 + tf32) + np.abs(y_ref) * ulp + 1e-30


# ----------------------------------------------------------------- a1: gemm
@pytest.mark.parametrize("case", doc("gemm_cases.json")["cases"], ids=lambda c: c[0])
def test_exact_engine_gemm_is_bit_identical(case):
    name, dt, acc = case[0], case[1], case[2]
    x, wt, bias = gemm_case_inputs(case)
    Y = gemm(Matrix2D(x, dt), Matrix2D(wt, dt), bias=bias, accum=Precision.from_tag(acc), engine="exact")
    assert sha(Y.data) == doc("gemm_cases.json")["Y_sha256"][name]


@pytest.mark.parametrize("case", [c for c in doc("gemm_cases.json")["cases"] if c[1] in
                                  ("int8", "binary16-emulated", "binary32") and c[2] != "binary64"],
                         ids=lambda c: c[0])
def test_tensor_engine_gemm_parity(case):
    name, dt, acc = case[0], case[1], case[2]
    x, wt, bias = gemm_case_inputs(case)
    Y = gemm(Matrix2D(x, dt), Matrix2D(wt, dt), bias=bias, accum=Precision.from_tag(acc), engine="tensor")
    ref = O.gemm(x, wt, bias, dt, None if dt == "int8" else acc)
    if dt == "int8":
        assert Y.data.tobytes() == np.asarray(ref, np.int32).tobytes()  # bit-exact
        assert sha(Y.data) == doc("gemm_cases.json")["Y_sha256"][name]
    else:
        err = np.abs(Y.widened() - np.asarray(ref, np.float64))
        assert (err <= _fp_tolerance(x, wt, bias, ref, dt)).all(), float(err.max())


# ------------------------------------------------- a3/a4/a5: checksum + verify
@pytest.mark.parametrize("meta", [m for m in doc("checksum.json") if "dtype" in m], ids=lambda m: m["key"])
def test_checksum_and_verify_bit_identical(meta):
    g = npz("checksum.npz")
    name, dt, p = meta["key"], meta["dtype"], meta["precision"]
    wt, x, y, bias = g[f"{name}__wt"], g[f"{name}__x"], g[f"{name}__y"], g[f"{name}__bias"]
    L = Mo.LayerSpec(0, "L0", "embed", wt.shape[0], wt.shape[1], x.shape[0], Matrix2D(wt, dt), np.asarray(bias))
    chk = G.offline_checksum(L, Precision.from_tag(p))
    assert chk.w_sum.tobytes() == g[f"{name}__w_sum"].tobytes()  # K2 bit-exact
    assert chk.bias_sum == meta["bias_sum"]
    summaries = {m["key"]: m for m in doc("checksum.json") if "max_discrepancy" in m}
    for stat in ("per_sample", "batch_mean"):
        key = f"{name}__{stat}"
        if key not in summaries:
            continue
        eps = None if dt == "int8" else G.EpsilonModel(0, 1e-5, 1.0, 0.99, -1e-3, 1e-3, 100,
                                                        Precision.from_tag(p), stat)
        ytag = "int32" if dt == "int8" else "binary64"
        out = G.verify_layer(Matrix2D(x, dt), Matrix2D(y, ytag, _trusted=True), chk, eps)
        want_d = g[f"{key}__d"]
        # bit-identical everywhere except NaN payloads, which are platform-defined
        # (x86 default NaN 0xFFC00000 vs CUDA canonical 0x7FFFFFFF in binary32 folds)
        nan = np.isnan(want_d) if want_d.dtype.kind == "f" else np.zeros(want_d.shape, bool)
        assert np.array_equal(np.isnan(out.d) if out.d.dtype.kind == "f" else nan, nan)
        assert out.d[~nan].tobytes() == want_d[~nan].tobytes()
        assert out.flagged == [int(i) for i in np.flatnonzero(g[f"{key}__flags"])]
        want = summaries[key]
        assert out.triggered == want["triggered"]
        assert out.max_discrepancy == want["max_discrepancy"] or (
            math.isinf(out.max_discrepancy) and math.isinf(want["max_discrepancy"]))


# ---------------------------------------------------------------- config 1
def test_cfg1_fp32_1024_exact_engine_bit_identical_with_1000_flips():
    c = doc("cfg1.json")
    x, wt, bias = cfg1_inputs(c["n"], c["seed"])
    X, Wt = Matrix2D(x, "binary32"), Matrix2D(wt, "binary32")
    Y = gemm(X, Wt, bias=bias, accum=Precision.BINARY32, engine="exact")
    assert sha(Y.data) == c["Y_sha256"]
    L = Mo.LayerSpec(0, "L0", "embed", c["n"], c["n"], c["n"], Wt, bias)
    chk = G.offline_checksum(L, Precision.BINARY64)
    assert sha(chk.w_sum) == c["w_sum_sha256"] and chk.bias_sum == c["bias_sum"]
    d = G._discrepancies(X.widened(), Y.widened(), chk)
    assert sha(d) == c["d_sha256"]
    mu, sigma, lo, hi = c["eps"]
    eps = G.EpsilonModel(0, mu, sigma, 0.9999, lo, hi, c["n"], Precision.BINARY64)
    y = Y.widened()
    for e, bit, trig, flagged, _ in c["flips"]:
        yc = y.copy()
        flat = yc.reshape(-1)
        flat[e] = float(I._flipped(float(np.float32(flat[e])), bit, "binary32"))
        out = G._verify_arrays(X.widened(), yc, chk, eps)
        assert int(out.triggered) == trig and out.flagged == flagged


def test_cfg1_default_engine_for_binary32_is_the_bit_exact_one():
    """binary32 models default to the bit-exact engine (Y, d and flags equal
    the reference's: the test above); the tensor pipe is an explicit opt-in."""
    from paper_2310_03841_b200.numerics import resolve_engine

    assert resolve_engine("binary32", Precision.BINARY32, None) == "exact"
    assert resolve_engine("binary16-emulated", Precision.BINARY32, None) == "tensor"
    assert resolve_engine("int8", Precision.INT64, None) == "tensor"
    assert resolve_engine("binary32", Precision.BINARY32, "tensor") == "tensor"


def test_cfg1_tensor_engine_3xtf32_detects_what_the_reference_detects():
    """Config 1 on the opt-in tensor path (binary32 as 3xTF32 + the fused
    check), calibrated the reference's way on its own clean rows (c = 0.9999).

    * Y within binary32 accuracy; the clean row-sum noise sigma within 5x of
      the reference's (the tensor core's truncating fp32 accumulator; plain
      TF32 is 1400x);
    * for each of the 1000 golden output flips, the injected row is flagged
      iff the reference flags it, except flips whose reference discrepancy
      falls between the two half-widths (widened by the per-row numerics
      band): the count of such flips is reported and bounded;
    * every other row's flag is its clean flag (rows are independent)."""
    import torch

    from paper_2310_03841_b200 import kernels as K

    c = doc("cfg1.json")
    n = c["n"]
    x, wt, bias = cfg1_inputs(n, c["seed"])
    X, Wt = Matrix2D(x, "binary32"), Matrix2D(wt, "binary32")
    Yref = gemm(X, Wt, bias=bias, accum=Precision.BINARY32, engine="exact")
    assert sha(Yref.data) == c["Y_sha256"]
    L = Mo.LayerSpec(0, "L0", "embed", n, n, n, Wt, bias)
    chk = G.offline_checksum(L, Precision.BINARY64)
    d_ref = G._discrepancies(X.widened(), Yref.widened(), chk)
    mu, sigma, lo, hi = c["eps"]
    xd = torch.from_numpy(x).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(wt.T)).cuda()
    bd = torch.from_numpy(bias.astype(np.float32)).cuda()
    w_split = K.split_tf32x3(wd, 1)
    base = dict(w_sum=chk.w_sum_device(), bias_sum=chk.bias_sum, w_split=w_split)
    y_t, res = K.protected_gemm(xd, wd, bd, lo=-1e300, hi=1e300, **base)
    y_t = y_t.cpu().numpy()
    d_t = res.d.cpu().numpy()
    ref_y = Yref.widened()
    mag = np.abs(x.astype(np.float64)) @ np.abs(wt.astype(np.float64)) + np.abs(bias)
    assert np.all(np.abs(y_t - ref_y) <= mag * (n * 2.0**-23 + 2.0**-20) + np.abs(ref_y) * 2.0**-23)
    e = O.fit_epsilon(d_t, 0.9999)
    mu_t, sig_t, lo_t, hi_t = e["mu"], e["sigma"], e["threshold_low"], e["threshold_high"]
    assert sig_t <= 5.0 * sigma, (sig_t, sigma)
    kw = dict(base, mu=mu_t, lo=lo_t, hi=hi_t)
    _, clean = K.protected_gemm(xd, wd, bd, **kw)
    clean_flags = clean.flags.cpu().numpy().astype(bool)
    band = np.abs(d_t - d_ref) + 1e-12
    gap, agree, missed = 0, 0, 0
    for e_, bit, trig, flagged, _ in c["flips"]:
        row, col = divmod(e_, n)
        _, r2 = K.protected_gemm(xd, wd, bd, injections=[K.Injection(row=row, col=col, bit=bit)], **kw)
        f = r2.flags.cpu().numpy().astype(bool)
        others = np.ones(n, bool)
        others[row] = False
        assert np.array_equal(f[others], clean_flags[others])
        o_ref = float(np.float32(ref_y[row, col]))
        dr = d_ref[row] - (float(I._flipped(o_ref, bit, "binary32")) - o_ref)  # the reference's trial d
        ref_flag = row in flagged
        if f[row] == ref_flag:
            agree += 1
            continue
        g = abs(dr - mu) if math.isfinite(dr) else math.inf
        inner, outer = min(hi - mu, hi_t - mu_t), max(hi - mu, hi_t - mu_t)
        assert inner - 2 * band[row] <= g <= outer + 2 * band[row] + abs(mu_t - mu), (row, bit, g, inner, outer)
        gap += 1
        missed += int(ref_flag and not f[row])
    print(f"cfg1 3xTF32: sigma {sig_t:.3e} vs reference {sigma:.3e}; {agree}/1000 injected-row flags equal, "
          f"{gap} inside the half-width gap ({missed} reference detections missed)")
    assert gap <= 60


def test_cfg1_tf32_opt_in_engine_is_single_pass_tf32():
    """Plain TF32 stays available as an explicit engine; it is narrower than
    binary32 (about 2^-11 per product), which is why it is not the default."""
    c = doc("cfg1.json")
    x, wt, bias = cfg1_inputs(c["n"], c["seed"])
    X, Wt = Matrix2D(x, "binary32"), Matrix2D(wt, "binary32")
    y32 = gemm(X, Wt, bias=bias, accum=Precision.BINARY32, engine="tensor").widened()
    y19 = gemm(X, Wt, bias=bias, accum=Precision.BINARY32, engine="tf32").widened()
    ref = gemm(X, Wt, bias=bias, accum=Precision.BINARY32, engine="exact").widened()
    e32, e19 = float(np.abs(y32 - ref).max()), float(np.abs(y19 - ref).max())
    assert e19 > 30 * e32, (e19, e32)


# ----------------------------------------------------- end-to-end toy pipelines
def _toy(docname):
    d = doc(docname)
    model = Mo.build_toy_model(*d["args"])
    ds = Mo.make_synthetic_dataset(model, *d["data"])
    return d, model, ds


def test_toy_int8_end_to_end_bit_identical():
    """int8 toy: weights, logits, golden set, ranges, epsilon, the detection
    campaign's CSV and summary, and the vulnerability campaign's CSV all equal
    the reference's bytes (tensor engine, fused checks)."""
    d, model, ds = _toy("toy_int8.json")
    assert [sha(L.weight.data) for L in model.layers] == d["weights_sha256"]
    assert [sha(np.asarray(L.bias)) for L in model.layers] == d["bias_sha256"]
    assert ds.labels == d["labels"]
    golden = Pr.select_golden(model, ds)
    assert golden.sample_ids == d["golden_ids"]
    ranges = Pr.profile_ranges(model, ds)
    assert {str(k): list(v) for k, v in ranges.bounds.items()} == d["ranges"]
    for x, want in zip(ds.inputs[:6], d["logits"]):
        assert Mo.forward(model, x, 0).logits.tolist() == want
    chks = {L.index: G.offline_checksum(L, Precision.INT64) for L in model.layers}
    eps = G.calibrate_epsilon(model, golden, confidence=0.9999)
    assert G.epsilon_models_to_dict(eps) == d["eps"]
    n_inj, seed = d["inject"]
    rep = G.evaluate_detection(model, golden, range(len(model.layers)), chks, eps, ranges, n_per_layer=n_inj,
                               seed=seed, clean_passes=d["clean"])
    assert rep.to_csv() == d["detection_csv"]
    assert rep.summary() == d["detection_summary"]
    camp = I.run_campaign(model, golden, ranges, n_per_layer=n_inj, seed=seed)
    assert camp.to_csv() == d["campaign_csv"]


@pytest.mark.parametrize("docname", ["toy_fp16.json", "toy_fp32.json"])
def test_toy_float_exact_engine_bit_identical(docname, exact_engine):
    """binary16-emulated / binary32 toys on the exact engine: every reference
    artifact reproduced byte for byte."""
    d, model, ds = _toy(docname)
    assert [sha(L.weight.data) for L in model.layers] == d["weights_sha256"]
    assert ds.labels == d["labels"]
    golden = Pr.select_golden(model, ds)
    assert golden.sample_ids == d["golden_ids"]
    ranges = Pr.profile_ranges(model, ds)
    assert {str(k): list(v) for k, v in ranges.bounds.items()} == d["ranges"]
    for x, want in zip(ds.inputs[:6], d["logits"]):
        assert Mo.forward(model, x, 0).logits.tolist() == want
    n_inj, seed = d["inject"]
    if "eps" in d:
        chks = {L.index: G.offline_checksum(L, Precision.BINARY64) for L in model.layers}
        eps = G.calibrate_epsilon(model, golden, confidence=0.9999)
        assert G.epsilon_models_to_dict(eps) == d["eps"]
        rep = G.evaluate_detection(model, golden, range(len(model.layers)), chks, eps, ranges, n_per_layer=n_inj,
                                   seed=seed, clean_passes=d["clean"])
        assert rep.to_csv() == d["detection_csv"]
        assert rep.summary() == d["detection_summary"]
    camp = I.run_campaign(model, golden, ranges, n_per_layer=n_inj, seed=seed)
    assert camp.to_csv() == d["campaign_csv"]


def test_toy_fp16_tensor_engine_statistics_match_reference():
    """Tensor engine (fused checks) on the fp16 toy: the same golden set, and
    epsilon models within the fp32-accumulation noise of the reference's."""
    d, model, ds = _toy("toy_fp16.json")
    golden = Pr.select_golden(model, ds)
    eps = G.calibrate_epsilon(model, golden, confidence=0.9999)
    for k, m in G.epsilon_models_to_dict(eps).items():
        ref = d["eps"][k]
        assert m["n"] == ref["n"]
        assert abs(m["sigma"] - ref["sigma"]) <= 0.25 * ref["sigma"] + 1e-6
        assert abs(m["mu"] - ref["mu"]) <= 0.5 * ref["sigma"] + 1e-6


def test_sampler_specs_identical_to_reference(exact_engine):
    """Injected-error map: sample_injection on the same (seed, layer, k) and
    the same clean trace draws the same element / mode / bit / value."""
    s = doc("sampler.json")
    model = Mo.build_toy_model(*s["model"])
    ds = Mo.make_synthetic_dataset(model, *s["data"])
    golden = Pr.select_golden(model, ds)
    ranges = Pr.profile_ranges(model, ds)
    for loc, modes, layer, k, sid, *want in s["cases"]:
        rng = I.injection_rng(11, layer, k)
        got_sid = golden.sample_ids[int(rng.integers(len(golden)))]
        assert got_sid == sid
        t = Mo.forward(model, golden.input_for(sid), golden.labels[sid], tap=[layer])
        try:
            spec = I.sample_injection(model, ranges, golden, rng, layer_index=layer, sample_id=sid,
                                      locations=(loc,), modes=tuple(modes) if modes else None, seed=11,
                                      clean_trace=t)
            assert [spec.element_index, spec.bit_index, spec.mode, spec.value] == want
        except Exception as e:  # noqa: BLE001
            assert want[0] == "error" and type(e).__name__ == want[1] and str(e) == want[2]
