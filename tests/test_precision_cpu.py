"""guard.choose_checksum_precision (guard.py:230-274) against the reference's own choices
on toy models and their reference range profiles (tests/golden/precision.json, made by
tests/golden/make_golden.py precision), including the binary64 fallback and its warning."""

import warnings

import pytest

from paper_2310_03841_b200 import guard as G
from paper_2310_03841_b200 import model as Mo
from paper_2310_03841_b200.profiler import RangeProfile
from tests.golden_io import doc


@pytest.mark.parametrize("case", doc("precision.json")["cases"],
                         ids=lambda c: f"{c['args'][5]}-d{c['args'][1]}-{c['label']}")
def test_choose_checksum_precision_equals_reference(case):
    model = Mo.build_toy_model(*case["args"])
    ranges = RangeProfile({int(k): tuple(v) for k, v in case["ranges"].items()})
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        got = G.choose_checksum_precision(model, ranges)
    assert {str(k): v.value for k, v in got.items()} == case["chosen"]
    assert [str(x.message) for x in w] == case["warnings"]
