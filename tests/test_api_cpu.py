"""CPU: host-side logic of the drop-in package that needs no GPU — types,
validation and messages, scalar encodings, thresholds, JSON/CSV artifacts —
plus the rule that the product path fails loudly without a CUDA device."""

import math

import numpy as np
import pytest

from paper_2310_03841_b200 import errors as E
from paper_2310_03841_b200.guard import (
    CorrectionPolicy,
    EpsilonModel,
    epsilon_models_from_json,
    epsilon_models_to_json,
    threshold_from_confidence,
)
from paper_2310_03841_b200.injector import (
    CampaignResult,
    InjectionRecord,
    InjectionSpec,
    bit_range,
    margin_of_error,
    merge_campaigns,
)
from paper_2310_03841_b200.numerics import Matrix2D, Precision, encoding_of, flip_bit, float_fields, round_to


def test_matrix_validation_messages():
    with pytest.raises(ValueError, match="2-D"):
        Matrix2D([1, 2, 3])
    with pytest.raises(ValueError, match="lattice"):
        Matrix2D([[1.0 + 2.0**-20]], "binary16-emulated")
    Matrix2D([[1.0 + 2.0**-10]], "binary16-emulated")
    with pytest.raises(ValueError):
        Matrix2D([[300]], "int8")
    with pytest.raises(ValueError):
        Matrix2D(np.zeros((0, 3)))
    assert Matrix2D([[0.0]]) != Matrix2D([[-0.0]])  # bytewise equality
    with pytest.raises(TypeError):
        hash(Matrix2D([[1.0]]))
    m = Matrix2D([[1, 2]], "int8")
    assert m.widened().dtype == np.int64 and m.copy() == m


def test_precision_and_fields():
    assert Precision.from_tag("int64-exact") is Precision.INT64
    assert [p.width for p in Precision] == [16, 32, 64, 64]
    assert Precision.BINARY16.accumulator_dtype == np.float16
    assert float_fields("binary16-emulated") == (10, 5)
    assert encoding_of("int32")[2] == 32
    with pytest.raises(ValueError):
        Precision.from_tag("binary8")


@pytest.mark.parametrize("dtype", ["binary64", "binary32", "binary16-emulated", "int8", "int32"])
def test_flip_bit_involution(dtype):
    sdt, udt, bits = encoding_of(dtype)
    vals = [sdt.type(v) for v in ((0.0, -1.5, 3.25, np.inf) if dtype.startswith("binary") else (0, -7, 100))]
    for v in vals:
        for i in range(bits):
            once = flip_bit(v, i, dtype)
            assert np.array([flip_bit(once, i, dtype)], sdt).tobytes() == np.array([v], sdt).tobytes()
    with pytest.raises(ValueError, match="bit index"):
        flip_bit(1.0, 64, "binary64")
    assert flip_bit(np.float32(1.0), 31, "binary32") == np.float32(-1.0)


def test_round_to_rules():
    assert round_to(65520.0, Precision.BINARY16) == math.inf
    assert round_to(2.0**-25, Precision.BINARY16) == 0.0
    assert math.isnan(round_to(math.nan, Precision.BINARY32))
    with pytest.raises(ValueError):
        round_to(1.0, Precision.INT64)


def test_thresholds_and_margin():
    lo, hi = threshold_from_confidence(0.0, 1.0, 0.9999)
    assert hi == pytest.approx(3.8906, abs=1e-4) and lo == -hi
    assert threshold_from_confidence(2.5, 0.0, 0.99) == (2.5, 2.5)
    with pytest.raises(ValueError):
        threshold_from_confidence(0.0, 1.0, 0.4)
    assert 0.00238 <= margin_of_error(102400, 0.9, 0.99) <= 0.00245
    assert margin_of_error(400, 0.5, 0.95) == pytest.approx(0.049, abs=5e-4)
    with pytest.raises(ValueError):
        margin_of_error(10, 0.5, 1.0)
    assert bit_range("binary32", "fp_sign_bit") == (31, 32)


def test_correction_policy_validation():
    with pytest.raises(ValueError):
        CorrectionPolicy("retry")
    with pytest.raises(ValueError):
        CorrectionPolicy("replay", max_replays=0)
    assert CorrectionPolicy("skip_to_head").max_replays == 3


def test_epsilon_json_round_trip():
    models = {i: EpsilonModel(i, 1e-6 * i, 0.5, 0.9999, -1.0, 1.0 + i, 100, Precision.BINARY64, "per_sample", 0.25)
              for i in range(3)}
    assert epsilon_models_from_json(epsilon_models_to_json(models)) == models


def _rec(layer, k, mismatch):
    spec = InjectionSpec(layer, "output", k, 3, "fp_mantissa_bit", 0, 7)
    return InjectionRecord(spec, 1.0, 1.5, 0.25, 0.5 + k, 1, 1 if not mismatch else 2, mismatch)


def test_campaign_csv_round_trip_and_merge():
    a = CampaignResult([_rec(0, 0, False), _rec(0, 1, True), _rec(2, 0, False)], 7, 2, {1: 2})
    text = a.to_csv()
    assert CampaignResult.from_csv(text, seed=7, n_per_layer=2).to_csv() == text
    s0 = CampaignResult([_rec(0, 0, False), _rec(0, 1, True), _rec(2, 0, False)], 7, 2, {})
    s1 = CampaignResult([], 7, 2, {1: 2})
    assert merge_campaigns([s0, s1]).to_csv() == text
    t = a.layer_tallies()
    assert t[0]["injections"] == 2 and t[0]["mismatches"] == 1


def test_error_hierarchy():
    for cls in (E.WeightFormatError, E.SamplingError, E.CalibrationError, E.GuardError, E.StageError,
                E.ConfigError):
        assert issubclass(cls, E.WorkbenchError)


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2310_03841_b200._lib import GemmGuardLibraryError
    from paper_2310_03841_b200.numerics import gemm

    with pytest.raises(GemmGuardLibraryError, match="CUDA"):
        gemm(Matrix2D([[1.0]]), Matrix2D([[1.0]]))


def test_checked_output_verdict_is_dropped_when_bytes_change():
    """a fused verdict must not survive an in-place edit of the
    output (a monkeypatched run_layer writing y[r, c] = bad, or a write through
    a reshape view as guard.py:517-521 does)."""
    from paper_2310_03841_b200.model import CheckedOutput

    y = np.arange(12, dtype=np.float64).reshape(3, 4).view(CheckedOutput).bind(("chk", "eps", "outcome"))
    assert y.fused_verdict() == ("chk", "eps", "outcome")
    y[1, 2] = 99.0
    assert y.fused_verdict() is None
    z = np.arange(12, dtype=np.int32).reshape(3, 4).view(CheckedOutput).bind(("c", "e", "o"))
    z.reshape(-1)[5] ^= 1 << 20  # write through a view
    assert z.fused_verdict() is None
    assert np.asarray(z).view(CheckedOutput).fused_verdict() is None  # derived arrays carry nothing
