"""Generate the golden fixtures of the parity tests by running the REFERENCE.

Imports the unmodified reference package from /root/reference/pkg/src (this
container only; /root/reference does not exist on the GPU box) and records
its outputs on seeded inputs:

  gemm.npz         numerics.gemm for every (dtype, accum) pair, incl. the
                   k-loop path (B*I*O > 2^26) and int32 wrap-around
  checksum.npz     guard.offline_checksum + guard.verify_layer (d, flags,
                   max_discrepancy, triggered) incl. NaN/Inf, batch_mean, int
  cfg1.json        config 1: fp32 1024^3 GEMM (sha256 of Y), its checksum,
                   verify on a calibrated epsilon and 1000 output flips
  toy_int8.json    an int8 toy pipeline end to end: weights hash, logits,
                   golden set, ranges, calibration, evaluate_detection records,
                   run_campaign CSV (bit-exact targets for the GPU path)
  toy_fp16.json    a binary16-emulated toy: weights hash, reference epsilon
                   models and detection summary (statistical targets)
  sampler.json     sample_injection specs for fixed traces / ranges / seeds

Run:  python tests/golden/make_golden.py      (writes next to this file)
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from gemmguard import guard as G  # noqa: E402
from gemmguard import injector as I  # noqa: E402
from gemmguard import model as Mo  # noqa: E402
from gemmguard import profiler as Pr  # noqa: E402
from gemmguard.numerics import Matrix2D, Precision, gemm  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand_matrix(rng, rows, cols, dtype):
    """Same generator as the GPU tests (tests/parity_inputs.py)."""
    if dtype == "int8":
        return Matrix2D(rng.integers(-128, 128, (rows, cols)), "int8")
    if dtype == "int32":
        return Matrix2D(rng.integers(-(2**20), 2**20, (rows, cols)), "int32")
    v = rng.standard_normal((rows, cols))
    if dtype == "binary16-emulated":
        v = v.astype(np.float16).astype(np.float64)
    elif dtype == "binary32":
        v = v.astype(np.float32)
    return Matrix2D(v, dtype)


GEMM_CASES = [
    # name, dtype, accum, B, I, O, seed
    ("f64_small", "binary64", "binary64", 5, 17, 7, 1),
    ("f32_f32", "binary32", "binary32", 33, 70, 45, 2),
    ("f32_f64", "binary32", "binary64", 9, 40, 12, 3),
    ("f16_f32", "binary16-emulated", "binary32", 37, 64, 50, 4),
    ("f16_f64", "binary16-emulated", "binary64", 8, 31, 9, 5),
    ("i8", "int8", "int64-exact", 40, 96, 72, 6),
    ("i8_bigk", "int8", "int64-exact", 3, 3072, 20, 7),
    ("i32_wrap", "int32", "int64-exact", 4, 9, 6, 8),
    ("f32_kloop", "binary32", "binary32", 64, 1100, 960, 9),  # B*I*O > 2^26: k-loop path
]


def make_gemm():
    arrs, hashes = {}, {}
    for name, dt, acc, B, Ii, O, seed in GEMM_CASES:
        rng = np.random.default_rng(seed)
        X = rand_matrix(rng, B, Ii, dt)
        Wt = rand_matrix(rng, Ii, O, dt)
        if dt in ("int8", "int32"):
            bias = rng.integers(-50, 50, O).astype(np.int32)
            if dt == "int32":
                bias = rng.integers(-(2**31), 2**31 - 1, O).astype(np.int64)  # wraps in astype(int32)
        else:
            bias = rand_matrix(rng, 1, O, dt).data[0].astype(np.float64)
        Y = gemm(X, Wt, bias=bias, accum=Precision.from_tag(acc))
        hashes[name] = sha(Y.data)
        if B * Ii * O > 1 << 20:
            continue  # large case: the test regenerates X, Wt, bias from the seed and compares sha256(Y)
        arrs[f"{name}__X"] = X.data
        arrs[f"{name}__Wt"] = Wt.data
        arrs[f"{name}__bias"] = bias
        arrs[f"{name}__Y"] = Y.data
    np.savez_compressed(OUT / "gemm.npz", **arrs)
    (OUT / "gemm_cases.json").write_text(json.dumps({"cases": GEMM_CASES, "Y_sha256": hashes}, indent=1))


def layer_from(wt, bias, dtype, index=0, tokens=2):
    w = Matrix2D(wt, dtype)
    return Mo.LayerSpec(index=index, name=f"L{index}", kind="embed", in_dim=w.rows, out_dim=w.cols, tokens=tokens,
                        weight=w, bias=np.asarray(bias))


def eps_model(lo, hi, mu=0.0, stat="per_sample", p=Precision.BINARY64):
    return G.EpsilonModel(layer_index=0, mu=mu, sigma=1.0, confidence=0.99, threshold_low=lo, threshold_high=hi,
                          n_samples=100, precision=p, statistic=stat)


def make_checksum():
    arrs, meta = {}, []
    rng = np.random.default_rng(21)
    cases = []
    # float layers, several checksum precisions
    for p in ("binary64", "binary32", "binary16-emulated"):
        for dt in ("binary32", "binary16-emulated", "binary64"):
            wt = rand_matrix(rng, 48, 40, dt)
            x = rand_matrix(rng, 30, 48, dt)
            bias = rand_matrix(rng, 1, 40, dt).data[0].astype(np.float64)
            cases.append((f"{dt}_{p}", dt, p, wt, x, bias))
    wt = rand_matrix(rng, 64, 50, "int8")
    x = rand_matrix(rng, 20, 64, "int8")
    cases.append(("int8_int64", "int8", "int64-exact", wt, x, rng.integers(-64, 65, 50).astype(np.int32)))
    for name, dt, p, wt, x, bias in cases:
        prec = Precision.from_tag(p)
        L = layer_from(wt.data, bias, dt, tokens=x.rows)
        chk = G.offline_checksum(L, prec)
        acc = Precision.INT64 if dt == "int8" else (Precision.BINARY64 if dt == "binary64" else Precision.BINARY32)
        Y = gemm(x, L.weight, bias=bias, accum=acc)
        y = Y.widened().copy()
        # corrupt a few rows so some flag; add NaN / Inf rows for floats
        y[3, 5] += 7.0 if dt != "int8" else 7
        if dt != "int8":
            y[4, 0] = np.nan
            y[6, 1] = np.inf
        Yc = Matrix2D(y, "int32" if dt == "int8" else ("binary64" if dt != "binary16-emulated" else "binary64"),
                      _trusted=True)
        for stat in ("per_sample", "batch_mean"):
            if dt == "int8" and stat == "batch_mean":
                continue
            eps = None if dt == "int8" else eps_model(-1e-3, 1e-3, mu=1e-5, stat=stat, p=prec)
            out = G.verify_layer(x, Yc, chk, eps)
            key = f"{name}__{stat}"
            arrs[f"{key}__d"] = out.d
            arrs[f"{key}__flags"] = np.isin(np.arange(x.rows), out.flagged)
            meta.append({"key": key, "max_discrepancy": out.max_discrepancy, "triggered": out.triggered})
        arrs[f"{name}__wt"] = wt.data
        arrs[f"{name}__x"] = x.data
        arrs[f"{name}__bias"] = bias
        arrs[f"{name}__y"] = y
        arrs[f"{name}__w_sum"] = chk.w_sum
        meta.append({"key": name, "dtype": dt, "precision": p, "bias_sum": chk.bias_sum})
    np.savez_compressed(OUT / "checksum.npz", **arrs)
    (OUT / "checksum.json").write_text(json.dumps(meta, indent=1))


def make_cfg1():
    """Config 1: fp32 1024^3 checksum-protected GEMM + 1000 output flips."""
    n = 1024
    rng = np.random.default_rng(np.random.SeedSequence(2310))
    x = rng.standard_normal((n, n)).astype(np.float32)
    wt = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    bias = (0.02 * rng.standard_normal(n)).astype(np.float32).astype(np.float64)
    X, Wt = Matrix2D(x, "binary32"), Matrix2D(wt, "binary32")
    Y = gemm(X, Wt, bias=bias, accum=Precision.BINARY32)
    L = layer_from(wt, bias, "binary32", tokens=n)
    chk = G.offline_checksum(L, Precision.BINARY64)
    d = G._discrepancies(X.widened(), Y.widened(), chk)
    lo, hi = G.threshold_from_confidence(float(d.mean()), float(d.std(ddof=1)), 0.9999)
    eps = G.EpsilonModel(0, float(d.mean()), float(d.std(ddof=1)), 0.9999, lo, hi, n, Precision.BINARY64)
    # 1000 output flips, default modes, seeded per flip like the campaigns
    y = Y.widened()
    flips = []
    for k in range(1000):
        r = np.random.default_rng(np.random.SeedSequence((2310, 0, k)))
        e = int(r.integers(y.size))
        mode = ("fp_exponent_bit", "fp_mantissa_bit")[int(r.integers(2))]
        b0, b1 = I._bit_range("binary32", mode)
        bit = int(r.integers(b0, b1))
        yc = y.copy()
        flat = yc.reshape(-1)
        orig = float(np.float32(flat[e]))
        flat[e] = float(I._flip(orig, bit, "binary32"))
        out = G._verify_arrays(X.widened(), yc, chk, eps)
        flips.append([e, bit, int(out.triggered), out.flagged, out.max_discrepancy if np.isfinite(out.max_discrepancy) else "inf"])
    doc = {"n": n, "seed": 2310, "Y_sha256": sha(Y.data), "w_sum_sha256": sha(chk.w_sum), "bias_sum": chk.bias_sum,
           "d_sha256": sha(d), "d_head": d[:8].tolist(), "eps": [eps.mu, eps.sigma, lo, hi],
           "Y_head": Y.data[0, :8].astype(np.float64).tolist(), "flips": flips,
           "detected": int(sum(f[2] for f in flips))}
    (OUT / "cfg1.json").write_text(json.dumps(doc))


def toy_doc(model, n_data, seed_data, n_inject, seed_inject, clean_passes, calibrate=True):
    ds = Mo.make_synthetic_dataset(model, n_data, seed=seed_data)
    golden = Pr.select_golden(model, ds)
    ranges = Pr.profile_ranges(model, ds)
    doc = {"weights_sha256": [sha(L.weight.data) for L in model.layers],
           "bias_sha256": [sha(np.asarray(L.bias)) for L in model.layers],
           "labels": ds.labels, "golden_ids": golden.sample_ids,
           "ranges": {str(k): list(v) for k, v in ranges.bounds.items()},
           "logits": [Mo.forward(model, x, 0).logits.tolist() for x in ds.inputs[:6]]}
    if calibrate:
        chks = {L.index: G.offline_checksum(L, Precision.INT64 if model.is_integer else Precision.BINARY64)
                for L in model.layers}
        eps = G.calibrate_epsilon(model, golden, confidence=0.9999)
        doc["eps"] = G.epsilon_models_to_dict(eps)
        rep = G.evaluate_detection(model, golden, range(len(model.layers)), chks, eps, ranges,
                                   n_per_layer=n_inject, seed=seed_inject, clean_passes=clean_passes)
        doc["detection_summary"] = rep.summary()
        doc["detection_csv"] = rep.to_csv()
        doc["specs"] = [[r.spec.layer_index, r.spec.location, r.spec.element_index, r.spec.bit_index, r.spec.mode,
                         r.spec.sample_id] for r in rep.records]
    camp = I.run_campaign(model, golden, ranges, n_per_layer=n_inject, seed=seed_inject)
    doc["campaign_csv"] = camp.to_csv()
    return doc


def make_toys():
    m8 = Mo.build_toy_model(blocks=2, dim=16, tokens=8, classes=6, seed=77, dtype="int8")
    (OUT / "toy_int8.json").write_text(json.dumps(
        {"args": [2, 16, 8, 6, 77, "int8"], "data": [24, 5], "inject": [6, 13], "clean": 8,
         **toy_doc(m8, 24, 5, 6, 13, 8)}))
    m16 = Mo.build_toy_model(blocks=1, dim=8, tokens=4, classes=5, seed=41, dtype="binary16-emulated")
    (OUT / "toy_fp16.json").write_text(json.dumps(
        {"args": [1, 8, 4, 5, 41, "binary16-emulated"], "data": [40, 4], "inject": [8, 3], "clean": 10,
         **toy_doc(m16, 40, 4, 8, 3, 10)}))
    m32 = Mo.build_toy_model(blocks=1, dim=12, tokens=5, classes=4, seed=9, dtype="binary32")
    (OUT / "toy_fp32.json").write_text(json.dumps(
        {"args": [1, 12, 5, 4, 9, "binary32"], "data": [12, 2], "inject": [3, 1], "clean": 4,
         **toy_doc(m32, 12, 2, 3, 1, 4, calibrate=False)}))


def make_sampler():
    """sample_injection on fixed traces: pure function of (rng stream, values, range)."""
    model = Mo.build_toy_model(blocks=1, dim=8, tokens=4, classes=5, seed=3, dtype="binary16-emulated")
    ds = Mo.make_synthetic_dataset(model, 12, seed=1)
    golden = Pr.select_golden(model, ds)
    ranges = Pr.profile_ranges(model, ds)
    out = []
    for loc in ("output", "input", "weight"):
        for modes in (None, ("fp_sign_bit",), ("random_value",), ("fp_exponent_bit", "fp_mantissa_bit", "fp_sign_bit")):
            for layer in range(len(model.layers)):
                for k in range(4):
                    rng = I._injection_rng(11, layer, k)
                    sid = golden.sample_ids[int(rng.integers(len(golden)))]
                    t = Mo.forward(model, golden.input_for(sid), golden.labels[sid], tap=[layer])
                    try:
                        s = I.sample_injection(model, ranges, golden, rng, layer_index=layer, sample_id=sid,
                                               locations=(loc,), modes=modes, seed=11, clean_trace=t)
                        out.append([loc, modes, layer, k, sid, s.element_index, s.bit_index, s.mode, s.value])
                    except Exception as e:  # SamplingError
                        out.append([loc, modes, layer, k, sid, "error", type(e).__name__, str(e), None])
    (OUT / "sampler.json").write_text(json.dumps({"model": [1, 8, 4, 5, 3, "binary16-emulated"], "data": [12, 1],
                                                  "cases": out}))


PRECISION_CASES = [  # build_toy_model args (blocks, dim, tokens, classes, seed, dtype), dataset (size, seed)
    ([1, 8, 4, 5, 3, "binary16-emulated"], [12, 1]),
    ([2, 16, 6, 4, 5, "binary16-emulated"], [10, 2]),
    ([1, 64, 8, 10, 7, "binary16-emulated"], [8, 3]),
    ([2, 32, 8, 6, 9, "binary32"], [8, 4]),
    ([1, 128, 4, 10, 11, "binary32"], [6, 5]),
    ([1, 8, 4, 5, 3, "int8"], [12, 1]),
]


def make_precision():
    """guard.choose_checksum_precision on toy models with the reference's own range profiles;
    plus a degenerate (near-zero span) profile that exhausts every precision (binary64 fallback + warning)."""
    import warnings

    cases = []
    for args, data in PRECISION_CASES:
        model = Mo.build_toy_model(*args)
        ds = Mo.make_synthetic_dataset(model, *data)
        ranges = Pr.profile_ranges(model, ds)
        for label, bounds in (("profiled", ranges.bounds),
                              ("narrow", {i: (lo, lo + 1e-30) for i, (lo, hi) in ranges.bounds.items()})):
            with warnings.catch_warnings(record=True) as w:
                warnings.simplefilter("always")
                got = G.choose_checksum_precision(model, Pr.RangeProfile(dict(bounds)))
            cases.append({"args": args, "ranges": {str(k): list(v) for k, v in bounds.items()}, "label": label,
                          "chosen": {str(k): v.value for k, v in got.items()},
                          "warnings": [str(x.message) for x in w]})
    (OUT / "precision.json").write_text(json.dumps({"cases": cases}, indent=1))


def make_albt():
    """weights_io.save_weights of two toy models: the ALBT fixtures of tests/test_albt_*.py."""
    from gemmguard import weights_io as W

    for name, args in (("toy_fp16.albt", [1, 8, 4, 5, 3, "binary16-emulated"]), ("toy_int8.albt", [2, 8, 4, 5, 7, "int8"]),
                       ("toy_fp32.albt", [1, 12, 5, 4, 9, "binary32"])):
        W.save_weights(OUT / name, Mo.build_toy_model(*args))
    (OUT / "albt.json").write_text(json.dumps({"toy_fp16.albt": [1, 8, 4, 5, 3, "binary16-emulated"],
                                               "toy_int8.albt": [2, 8, 4, 5, 7, "int8"],
                                               "toy_fp32.albt": [1, 12, 5, 4, 9, "binary32"]}))


if __name__ == "__main__":
    import numpy

    parts = sys.argv[1:] or ["gemm", "checksum", "sampler", "toys", "cfg1", "precision", "albt"]
    for part in parts:
        {"gemm": make_gemm, "checksum": make_checksum, "sampler": make_sampler, "toys": make_toys,
         "cfg1": make_cfg1, "precision": make_precision, "albt": make_albt}[part]()
    (OUT / "VERSIONS.json").write_text(json.dumps({"numpy": numpy.__version__, "python": sys.version.split()[0],
                                                    "reference": str(REF)}))
    print("golden fixtures written to", OUT)
