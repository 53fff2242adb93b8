"""ALBT v1 container (weights_io.py:1-7) against files written by the reference's
save_weights (tests/golden/*.albt, tests/golden/make_golden.py albt): the graph and
weights read back exactly, our writer reproduces the reference's bytes, and the
reference's format errors are raised."""

import pytest

from paper_2310_03841_b200 import albt
from paper_2310_03841_b200 import model as Mo
from paper_2310_03841_b200.errors import WeightFormatError
from tests.golden_io import GOLDEN, doc


@pytest.mark.parametrize("name", sorted(doc("albt.json")))
def test_albt_round_trip_is_the_references(name, tmp_path):
    args = doc("albt.json")[name]
    ref = Mo.build_toy_model(*args)
    got = albt.load_model(GOLDEN / name)
    assert (got.dtype, got.tokens, got.num_classes, got.input_dim, got.seed) == \
        (ref.dtype, ref.tokens, ref.num_classes, ref.input_dim, ref.seed)
    for a, b in zip(got.layers, ref.layers):
        assert (a.kind, a.in_dim, a.out_dim, a.tokens, a.activation, a.normalize_before) == \
            (b.kind, b.in_dim, b.out_dim, b.tokens, b.activation, b.normalize_before)
        assert a.weight == b.weight and a.bias.tobytes() == b.bias.tobytes()
    out = tmp_path / name
    albt.save(out, got)
    assert out.read_bytes() == (GOLDEN / name).read_bytes()


def test_albt_format_errors(tmp_path):
    blob = (GOLDEN / "toy_fp16.albt").read_bytes()
    for bad, msg in ((b"XXXX" + blob[4:], "magic"), (blob[:4] + b"\x02" + blob[5:], "version"),
                     (blob[:40], "truncated")):
        p = tmp_path / "bad.albt"
        p.write_bytes(bad)
        with pytest.raises(WeightFormatError, match=msg):
            albt.load_model(p)
