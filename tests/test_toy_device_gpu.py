"""GPU: the batched device forward of the integer toy
equals the reference byte for byte — logits of the golden fixture, the host
path's per-sample logits, and profile_ranges computed on the device."""

import numpy as np
import pytest

from paper_2310_03841_b200 import model as Mo
from paper_2310_03841_b200 import toy_device as TD
from tests.golden_io import doc

pytestmark = pytest.mark.gpu


def _toy():
    d = doc("toy_int8.json")
    model = Mo.build_toy_model(*d["args"])
    ds = Mo.make_synthetic_dataset(model, *d["data"])
    return d, model, ds


def test_batched_device_forward_matches_reference_logits_and_ranges():
    d, model, ds = _toy()
    ranges = {}
    out = TD.forward_batch(model, ds.inputs, ds.labels, ranges=ranges)
    for i, want in enumerate(d["logits"]):
        assert out.logits[i].tolist() == want
    for i, x in enumerate(ds.inputs):
        ref = Mo.forward(model, x, ds.labels[i])
        assert out.logits[i].tolist() == ref.logits.tolist()
        assert out.predicted[i] == ref.predicted_class
        assert out.losses[i] == ref.loss
    got = {str(k): [r.bounds()[0], r.bounds()[1]] for k, r in ranges.items()}
    assert got == d["ranges"]
    assert all(r.bounds()[2] == 0 for r in ranges.values())


def test_batched_device_forward_protected_is_clean_and_batch_invariant():
    d, model, ds = _toy()
    full = TD.forward_batch(model, ds.inputs, protect=True)
    assert all(not f.any() for f in full.flagged.values())
    part = TD.forward_batch(model, ds.inputs[3:9], protect=True)
    assert np.array_equal(part.logits, full.logits[3:9])


def test_float_models_stay_on_the_host_path():
    model = Mo.build_toy_model(1, 16, 4, 3, 0, "binary32")
    ds = Mo.make_synthetic_dataset(model, 2, 0)
    with pytest.raises(NotImplementedError):
        TD.forward_batch(model, ds.inputs)
