"""The workbench CLI on the host: config validation and exit codes,
the config-hash / seeds stamps, and the host stages (analyze, plan, report) reproducing the
reference's artifact bytes from the reference's upstream artifacts
(tests/golden/cli/*, written by tests/golden/make_cli_golden.py)."""

from __future__ import annotations

import json
import shutil
import warnings
from pathlib import Path

import pytest

from paper_2310_03841_b200.cli import STAGES, WorkbenchConfig, main

GOLDEN = Path(__file__).parent / "golden" / "cli"
NAMES = sorted(p.name for p in GOLDEN.iterdir())


def _config(tmp_path: Path, **over) -> Path:
    cfg = json.loads((GOLDEN / "fp16_toy" / "config.json").read_text())
    cfg.update(over)
    cfg["output_dir"] = str(tmp_path / "out")
    path = tmp_path / "config.json"
    path.write_text(json.dumps(cfg))
    return path


def test_stage_names_match_reference():
    assert STAGES == ("profile", "inject", "analyze", "calibrate", "plan", "evaluate", "report")


@pytest.mark.parametrize("name", NAMES)
def test_config_hash_and_seeds_match_reference_stamps(name):
    cfg = WorkbenchConfig.from_file(str(GOLDEN / name / "config.json"))
    doc = json.loads((GOLDEN / name / "ranges.json").read_text())
    assert cfg.config_hash() == doc["config_hash"]
    assert cfg.seeds() == doc["seeds"]


def test_missing_config_is_config_error(tmp_path):
    assert main(["profile", "--config", str(tmp_path / "nope.json")]) == 2


@pytest.mark.parametrize("raw, msg", [
    ("{not json", "not valid JSON"),
    ('{"model": {}}', "missing required section"),
    ('{"model": {"blocks": 1}, "dataset": {"size": 1, "seed": 1}, "campaign": {"n_per_layer": 1, "seed": 1},'
     ' "output_dir": "o"}', "synthetic model spec missing 'dim'"),
    ('{"model": {"path": "/nonexistent.albt"}, "dataset": {"size": 1, "seed": 1},'
     ' "campaign": {"n_per_layer": 1, "seed": 1}, "output_dir": "o"}', "model weights not found"),
    ('{"model": {"blocks": 1, "dim": 8, "tokens": 4, "classes": 5, "seed": 1}, "dataset": {"size": 1},'
     ' "campaign": {"n_per_layer": 1, "seed": 1}, "output_dir": "o"}', "dataset spec missing 'seed'"),
])
def test_invalid_config_is_config_error(tmp_path, capsys, raw, msg):
    bad = tmp_path / "bad.json"
    bad.write_text(raw)
    assert main(["profile", "--config", str(bad)]) == 2
    assert msg in capsys.readouterr().err


@pytest.mark.parametrize("stage, producer", [("inject", "profile"), ("calibrate", "profile"), ("analyze", "inject"),
                                             ("plan", "analyze"), ("evaluate", "calibrate"), ("report", "analyze")])
def test_stage_without_upstream_is_stage_error(tmp_path, capsys, stage, producer):
    assert main([stage, "--config", str(_config(tmp_path))]) == 3
    assert f"run the `{producer}` stage first" in capsys.readouterr().err


@pytest.mark.parametrize("name", NAMES)
def test_host_stages_reproduce_reference_bytes(tmp_path, name):
    """analyze -> plan -> report over the reference's own campaign / detection artifacts."""
    out = tmp_path / "out"
    out.mkdir()
    for upstream in ("campaign.csv", "campaign_summary.json", "detection_summary.json"):
        shutil.copy(GOLDEN / name / upstream, out / upstream)
    cfg = GOLDEN / name / "config.json"
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        for stage in ("analyze", "plan", "report"):
            assert main([stage, "--config", str(cfg), "--out", str(out)]) == 0, stage
    for artifact in ("vulnerability.json", "curve_duplication.csv", "curve_checksum.csv", "plan.json", "report.json"):
        assert (out / artifact).read_bytes() == (GOLDEN / name / artifact).read_bytes(), artifact


def test_seed_override_changes_the_hash(tmp_path):
    path = _config(tmp_path)
    a = WorkbenchConfig.from_file(str(path))
    out = tmp_path / "o2"
    out.mkdir()
    shutil.copy(GOLDEN / "fp16_toy" / "campaign.csv", out / "campaign.csv")
    assert main(["analyze", "--config", str(path), "--out", str(out), "--seed", "99"]) == 0
    stamped = json.loads((out / "vulnerability.json").read_text())
    assert stamped["seeds"]["campaign"] == 99 and stamped["config_hash"] != a.config_hash()


def test_env_overrides_output_dir(tmp_path, monkeypatch):
    path = _config(tmp_path)
    env_dir = tmp_path / "env_out"
    env_dir.mkdir()
    shutil.copy(GOLDEN / "fp16_toy" / "campaign.csv", env_dir / "campaign.csv")
    monkeypatch.setenv("GEMMGUARD_OUT", str(env_dir))
    assert main(["analyze", "--config", str(path)]) == 0
    assert (env_dir / "vulnerability.json").exists() and not (tmp_path / "out" / "vulnerability.json").exists()
