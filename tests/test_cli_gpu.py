"""The workbench CLI on the B200 backend: all seven stages of three
configs reproduce, byte for byte, the artifacts the reference CLI wrote for the same configs
(tests/golden/cli/*: ranges, golden set, campaign CSV, epsilon models, plan, detection
records, thresholds and the report), reruns are byte-identical (the config-hash determinism
contract, reference tests/test_cli.py:93-103), and a model loads from an ALBT weights file."""

from __future__ import annotations

import json
import warnings
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

pytest.importorskip("torch")

from paper_2310_03841_b200.cli import STAGES, main  # noqa: E402

GOLDEN = Path(__file__).parent / "golden" / "cli"
NAMES = sorted(p.name for p in GOLDEN.iterdir())


def _run_all(cfg: Path, out: Path, *extra: str) -> None:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        for stage in STAGES:
            assert main([stage, "--config", str(cfg), "--out", str(out), *extra]) == 0, stage


@pytest.mark.parametrize("name", NAMES)
def test_pipeline_reproduces_reference_artifacts(tmp_path, name):
    out = tmp_path / "out"
    _run_all(GOLDEN / name / "config.json", out)
    want = {p.name for p in (GOLDEN / name).iterdir()} - {"config.json"}
    assert {p.name for p in out.iterdir()} == want
    differ = [a for a in sorted(want) if (out / a).read_bytes() != (GOLDEN / name / a).read_bytes()]
    assert differ == []
    # determinism: a second run into another directory is byte-identical
    out2 = tmp_path / "out2"
    _run_all(GOLDEN / name / "config.json", out2)
    assert all((out / a).read_bytes() == (out2 / a).read_bytes() for a in want)


def test_evaluate_before_calibrate_is_stage_error(tmp_path, capsys):
    cfg = GOLDEN / "fp16_toy" / "config.json"
    assert main(["profile", "--config", str(cfg), "--out", str(tmp_path)]) == 0
    assert main(["evaluate", "--config", str(cfg), "--out", str(tmp_path)]) == 3
    assert "calibrate" in capsys.readouterr().err


def test_seed_flag_changes_the_campaign(tmp_path):
    cfg = GOLDEN / "int8_toy" / "config.json"
    for stage in ("profile", "inject"):
        assert main([stage, "--config", str(cfg), "--out", str(tmp_path / "alt"), "--seed", "99"]) == 0
    alt = (tmp_path / "alt" / "campaign.csv").read_text().splitlines()[1:]
    base = (GOLDEN / "int8_toy" / "campaign.csv").read_text().splitlines()[1:]
    assert alt != base and len(alt) == len(base)


def test_model_from_weights_file(tmp_path):
    from paper_2310_03841_b200 import albt
    from paper_2310_03841_b200.model import build_toy_model

    spec = json.loads((GOLDEN / "int8_toy" / "config.json").read_text())
    m = spec["model"]
    model = build_toy_model(blocks=m["blocks"], dim=m["dim"], tokens=m["tokens"], classes=m["classes"],
                            seed=m["seed"], dtype=m["dtype"])
    wpath = tmp_path / "weights.albt"
    albt.save(wpath, model)
    spec["model"] = {"path": str(wpath)}
    cfg = tmp_path / "config.json"
    cfg.write_text(json.dumps(spec))
    assert main(["profile", "--config", str(cfg), "--out", str(tmp_path / "o")]) == 0
    got = json.loads((tmp_path / "o" / "ranges.json").read_text())
    want = json.loads((GOLDEN / "int8_toy" / "ranges.json").read_text())
    assert got["ranges"] == want["ranges"]  # same weights, same ranges; only the stamp differs
    assert len(json.loads((tmp_path / "o" / "v_orig.json").read_text())["v_orig"]) == len(model.layers)


def test_tensor_engine_moves_only_low_bits(tmp_path):
    """--engine tensor (binary16 layers on tcgen05, fp32 accumulation in the tensor core's
    order): every artifact but the float discrepancies / epsilon models is the reference's
    bytes, detection flags included; the floats agree to 1e-3 of sigma."""
    name = "fp16_toy"
    out = tmp_path / "out"
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        for stage in STAGES:
            assert main([stage, "--config", str(GOLDEN / name / "config.json"), "--out", str(out),
                         "--engine", "tensor"]) == 0, stage
    floaty = {"epsilon.json", "thresholds.csv", "detection.csv"}
    for a in sorted({p.name for p in (GOLDEN / name).iterdir()} - {"config.json"} - floaty):
        assert (out / a).read_bytes() == (GOLDEN / name / a).read_bytes(), a
    got = json.loads((out / "epsilon.json").read_text())["epsilon"]
    want = json.loads((GOLDEN / name / "epsilon.json").read_text())["epsilon"]
    assert got.keys() == want.keys()
    for k in want:
        s = want[k]["sigma"]
        for f in ("mu", "sigma", "threshold_low", "threshold_high"):
            assert abs(got[k][f] - want[k][f]) <= 1e-3 * s, (k, f)
    rows = lambda p: [ln.split(",") for ln in p.read_text().splitlines()[2:]]  # noqa: E731
    g, w = rows(out / "detection.csv"), rows(GOLDEN / name / "detection.csv")
    assert [(r[0], r[2], r[3]) for r in g] == [(r[0], r[2], r[3]) for r in w]  # layer, mismatch, detected
    for rg, rw in zip(g, w):
        if rw[1]:
            assert abs(float(rg[1]) - float(rw[1])) <= 1e-6 + 1e-3 * abs(float(rw[1]))


def test_inject_with_workers_matches_single_process(tmp_path):
    """--workers 2 runs the float toy's layers in spawned worker processes (each its own CUDA
    context); the campaign CSV is the reference's single-process bytes."""
    cfg = GOLDEN / "fp16_toy" / "config.json"
    assert main(["profile", "--config", str(cfg), "--out", str(tmp_path)]) == 0
    assert main(["inject", "--config", str(cfg), "--out", str(tmp_path), "--workers", "2"]) == 0
    for a in ("campaign.csv", "campaign_summary.json"):
        assert (tmp_path / a).read_bytes() == (GOLDEN / "fp16_toy" / a).read_bytes(), a
