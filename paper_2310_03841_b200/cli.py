"""Workbench command line on the B200 backend.

The reference's batch front-end (/root/reference/pkg/src/gemmguard/cli.py)
with its stages pointed at this package: the same seven subcommands, the same
JSON config and defaults (cli.py:44-137), the same artifact names and bytes
(every artifact carries the config hash and the seeds, cli.py:147-155), the
same exit codes (0 ok, 2 config error, 3 missing upstream stage, 4 runtime
numerical error; cli.py:369-390) and the same overrides (`--out`,
`GEMMGUARD_OUT`, `--workers` / `GEMMGUARD_WORKERS`, `--seed`).

What runs on the device: `profile` (min/max ranges and the golden set from
device forwards), `inject` (the stratified campaign; integer models as
batched device forwards), `calibrate` (the device calibration of
`guard.calibrate_epsilon`) and `evaluate` (`guard.evaluate_detection` with the
fused check).  `analyze`, `plan` and `report` are host arithmetic over the
tallies (`planning.py`).  A config that runs through the reference CLI
produces the same artifact bytes here (`tests/test_cli_gpu.py`, against
artifacts the reference wrote: `tests/golden/make_cli_golden.py`).

The GEMMs run on the device's exact engine unless `--engine` or
$GEMMGUARD_ENGINE names another: the exact engine keeps the reference's
binary32 accumulation order, so float discrepancies, epsilon models and
thresholds are the reference's bytes; `--engine tensor` runs binary16 layers
on tcgen05 and moves only the low bits of those floats (flags unchanged on
the golden configs).

    python -m paper_2310_03841_b200.cli STAGE --config CONFIG.json [--out DIR] [--workers N] [--seed S]
                                              [--engine auto|tensor|exact|tf32]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
from contextlib import contextmanager
from dataclasses import dataclass
from pathlib import Path

from .errors import ConfigError, StageError, WorkbenchError
from .numerics import ENGINES

__all__ = ["STAGES", "WorkbenchConfig", "build_parser", "main"]

STAGES = ("profile", "inject", "analyze", "calibrate", "plan", "evaluate", "report")

GUARD_DEFAULTS = {"confidence": 0.9999, "precision": "auto", "target_coverage": 0.99, "per_sample": True}
CORRECTION_DEFAULTS = {"kind": "replay", "max_replays": 3}

# required keys per config section (cli.py:79-95); a model is either a weights file or a synthetic spec
_SYNTHETIC_MODEL = ("blocks", "dim", "tokens", "classes", "seed")
_SECTION_KEYS = {"dataset": ("size", "seed"), "campaign": ("n_per_layer", "seed")}


@dataclass
class WorkbenchConfig:
    """A validated workbench config; seeds are always explicit (cli.py:55-137)."""

    model: dict
    dataset: dict
    campaign: dict
    guard: dict
    correction: dict
    output_dir: str
    raw: dict

    @classmethod
    def from_file(cls, path: str) -> "WorkbenchConfig":
        try:
            text = Path(path).read_text()
        except OSError as exc:
            raise ConfigError(f"cannot read config {path}: {exc}") from exc
        try:
            raw = json.loads(text)
        except json.JSONDecodeError as exc:
            raise ConfigError(f"config {path} is not valid JSON: {exc}") from exc
        return cls.from_dict(raw)

    @classmethod
    def from_dict(cls, raw: dict) -> "WorkbenchConfig":
        missing = [k for k in ("model", "dataset", "campaign", "output_dir") if k not in raw]
        if missing:
            raise ConfigError(f"config missing required section {missing[0]!r}")
        model = raw["model"]
        if "path" in model:
            if not Path(model["path"]).exists():
                raise ConfigError(f"model weights not found: {model['path']}")
        else:
            gap = [k for k in _SYNTHETIC_MODEL if k not in model]
            if gap:
                raise ConfigError(f"synthetic model spec missing {gap[0]!r}")
        for section, keys in _SECTION_KEYS.items():
            gap = [k for k in keys if k not in raw[section]]
            if gap:
                raise ConfigError(f"{section} spec missing {gap[0]!r}")
        return cls(model=model, dataset=raw["dataset"], campaign=raw["campaign"],
                   guard={**GUARD_DEFAULTS, **raw.get("guard", {})},
                   correction={**CORRECTION_DEFAULTS, **raw.get("correction", {})},
                   output_dir=raw["output_dir"], raw=raw)

    def config_hash(self) -> str:
        """First 16 hex digits of the SHA-256 of the canonical raw config (cli.py:108-110)."""
        canon = json.dumps(self.raw, sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(canon.encode()).hexdigest()[:16]

    def seeds(self) -> dict:
        return {"model": self.model.get("seed"), "dataset": self.dataset["seed"], "campaign": self.campaign["seed"]}

    def build_model(self):
        if "path" in self.model:
            from .albt import load_model

            return load_model(self.model["path"])
        from .model import build_toy_model

        m = self.model
        return build_toy_model(blocks=m["blocks"], dim=m["dim"], tokens=m["tokens"], classes=m["classes"],
                               seed=m["seed"], dtype=m.get("dtype", "binary32"))

    def dataset_for(self, model):
        from .model import make_synthetic_dataset

        return make_synthetic_dataset(model, self.dataset["size"], self.dataset["seed"])

    def build_golden(self, model):
        from .profiler import select_golden

        return select_golden(model, self.dataset_for(model))

    def campaign_modes(self) -> tuple[str, ...] | None:
        modes = self.campaign.get("modes")
        return tuple(modes) if modes else None


class Artifacts:
    """The output directory: stamped writers and upstream-artifact readers (cli.py:140-174)."""

    def __init__(self, cfg: WorkbenchConfig, override: str | None):
        self.cfg = cfg
        self.dir = Path(override or os.environ.get("GEMMGUARD_OUT") or cfg.output_dir)
        self.dir.mkdir(parents=True, exist_ok=True)

    def write_json(self, name: str, doc: dict) -> None:
        stamped = {"config_hash": self.cfg.config_hash(), "seeds": self.cfg.seeds()}
        stamped.update(doc)
        (self.dir / name).write_text(json.dumps(stamped, indent=2, sort_keys=True) + "\n")

    def write_csv(self, name: str, text: str) -> None:
        seeds = json.dumps(self.cfg.seeds(), sort_keys=True, separators=(",", ":"))
        (self.dir / name).write_text(f"# config_hash={self.cfg.config_hash()} seeds={seeds}\n{text}")

    def need(self, name: str, producer: str) -> Path:
        path = self.dir / name
        if not path.exists():
            raise StageError(f"missing artifact {name}: run the `{producer}` stage first")
        return path

    def payload(self, name: str, producer: str, key: str):
        return json.loads(self.need(name, producer).read_text())[key]

    def csv_body(self, name: str, producer: str) -> str:
        lines = self.need(name, producer).read_text().splitlines(keepends=True)
        return "".join(ln for ln in lines if not ln.startswith("#"))

    def ranges(self):
        from .profiler import RangeProfile

        return RangeProfile.from_dict(self.payload("ranges.json", "profile", "ranges"))


# ------------------------------------------------------------------ stages


def stage_profile(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """ranges.json, golden.json, v_orig.json (cli.py:177-199)."""
    from .planning import compute_v_orig
    from .profiler import profile_ranges, select_golden

    model = cfg.build_model()
    data = cfg.dataset_for(model)
    ranges = profile_ranges(model, data)
    golden = select_golden(model, data)
    art.write_json("ranges.json", {"ranges": ranges.to_dict()})
    art.write_json("golden.json", {"golden": {"sample_ids": golden.sample_ids,
                                              "labels": {str(k): v for k, v in golden.labels.items()},
                                              "losses": {str(k): v for k, v in golden.losses.items()}}})
    share = compute_v_orig(model)
    art.write_json("v_orig.json", {"v_orig": {str(layer.index): float(share[layer.index]) for layer in model.layers}})


def stage_inject(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """campaign.csv, campaign_summary.json (cli.py:202-218)."""
    from .injector import run_campaign

    art.need("golden.json", "profile")
    ranges = art.ranges()
    model = cfg.build_model()
    result = run_campaign(model, cfg.build_golden(model), ranges, cfg.campaign["n_per_layer"],
                          modes=cfg.campaign_modes(), locations=tuple(cfg.campaign.get("locations", ["output"])),
                          seed=cfg.campaign["seed"], workers=workers)
    art.write_csv("campaign.csv", result.to_csv())
    art.write_json("campaign_summary.json", json.loads(result.summary_json()))


def stage_analyze(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """vulnerability.json and the two coverage curves, head reported apart (cli.py:221-253)."""
    from .injector import CampaignResult
    from . import planning as P

    result = CampaignResult.from_csv(art.csv_body("campaign.csv", "inject"), seed=cfg.campaign["seed"],
                                     n_per_layer=cfg.campaign["n_per_layer"])
    model = cfg.build_model()
    vul = P.layer_vulnerabilities(model, result)
    art.write_json("vulnerability.json", {"layers": [
        {"layer": x.layer_index, "v_orig": x.v_orig, "p_prop": x.p_prop, "delta_loss": x.delta_loss,
         "v_layer": x.v_layer} for x in vul]})
    flops, _ = P.model_totals(model)
    head = model.layers[-1].index
    body = [x for x in vul if x.layer_index != head]
    share = [x.v_layer for x in body]
    for name, cost_model in (("duplication", P.duplication_cost_model), ("checksum", P.checksum_cost_model)):
        cost = [cost_model(model.layers[x.layer_index])[0] / flops for x in body]
        art.write_csv(f"curve_{name}.csv", P.build_coverage_curve(share, cost).to_csv())


def stage_calibrate(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """epsilon.json from device calibration over the golden set (cli.py:256-273)."""
    from .guard import calibrate_epsilon, choose_checksum_precision, epsilon_models_to_dict
    from .numerics import Precision

    art.need("golden.json", "profile")
    ranges = art.ranges()
    model = cfg.build_model()
    golden = cfg.build_golden(model)
    tag = cfg.guard["precision"]
    if tag == "auto":
        precisions = choose_checksum_precision(model, ranges)
    else:
        fixed = Precision.from_tag(tag)
        precisions = {layer.index: fixed for layer in model.layers}
    eps = calibrate_epsilon(model, golden, precisions=precisions, confidence=cfg.guard["confidence"],
                            per_sample=cfg.guard["per_sample"])
    art.write_json("epsilon.json", {"epsilon": epsilon_models_to_dict(eps)})


def stage_plan(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """plan.json: checksum scheme, head forced in (cli.py:276-291)."""
    from . import planning as P

    rows = art.payload("vulnerability.json", "analyze", "layers")
    model = cfg.build_model()
    flops, mem = P.model_totals(model)
    costs = [P.checksum_cost_model(layer) for layer in model.layers]
    plan = P.select_layers([r["v_layer"] for r in rows], [c[0] for c in costs], cfg.guard["target_coverage"],
                           head_index=model.layers[-1].index, scheme="checksum", total_compute=flops,
                           memory_costs=[c[1] for c in costs], total_memory=mem)
    art.write_json("plan.json", {"plan": plan.to_dict()})


def stage_evaluate(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """detection.csv, thresholds.csv, detection_summary.json (cli.py:294-314)."""
    from .guard import epsilon_models_from_dict, evaluate_detection, offline_checksum
    from .planning import ProtectionPlan

    eps = epsilon_models_from_dict(art.payload("epsilon.json", "calibrate", "epsilon"))
    plan = ProtectionPlan.from_dict(art.payload("plan.json", "plan", "plan"))
    ranges = art.ranges()
    model = cfg.build_model()
    golden = cfg.build_golden(model)
    chks = {i: offline_checksum(model.layers[i], eps[i].precision) for i in eps}
    report = evaluate_detection(model, golden, plan, chks, eps, ranges, n_per_layer=cfg.campaign["n_per_layer"],
                                modes=cfg.campaign_modes(), seed=cfg.campaign["seed"])
    art.write_csv("detection.csv", report.to_csv())
    art.write_csv("thresholds.csv", report.thresholds_csv())
    art.write_json("detection_summary.json", {"detection": report.summary()})


def stage_report(cfg: WorkbenchConfig, art: Artifacts, workers: int) -> None:
    """report.json from the upstream artifacts (cli.py:317-340)."""
    from .injector import margin_of_error

    rows = art.payload("vulnerability.json", "analyze", "layers")
    campaign = art.payload("campaign_summary.json", "inject", "layers")
    plan = art.payload("plan.json", "plan", "plan")
    detection = art.payload("detection_summary.json", "evaluate", "detection")
    n = sum(v["injections"] for v in campaign.values())
    art.write_json("report.json", {
        "overall_sdc_probability": sum(r["v_layer"] for r in rows),
        "most_vulnerable_layer": max(rows, key=lambda r: r["v_layer"])["layer"],
        "zero_propagation_layers": [r["layer"] for r in rows if r["p_prop"] == 0.0],
        "head_p_prop": rows[-1]["p_prop"],
        "campaign_injections": n,
        "campaign_margin_of_error": margin_of_error(n, 0.9, 0.99) if n else None,
        "protection": plan,
        "detection": detection,
    })


STAGE_FNS = {name: globals()[f"stage_{name}"] for name in STAGES}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="gemmguard",
                                     description="Fault-injection and checksum-protection workbench for GEMM "
                                                 "pipelines (B200 backend)")
    sub = parser.add_subparsers(dest="stage", required=True)
    for name in STAGES:
        sp = sub.add_parser(name, help=f"run the {name} stage")
        sp.add_argument("--config", required=True, help="workbench config JSON")
        sp.add_argument("--out", default=None, help="output directory (overrides config)")
        sp.add_argument("--workers", type=int, default=None, help="campaign worker count")
        sp.add_argument("--seed", type=int, default=None, help="override the campaign seed")
        sp.add_argument("--engine", choices=ENGINES, default=None,
                        help="GEMM engine (default: $GEMMGUARD_ENGINE, else exact)")
    return parser


@contextmanager
def _engine(name: str | None):
    """Run a stage with GEMMGUARD_ENGINE = name (or its current value, else "exact")."""
    old = os.environ.get("GEMMGUARD_ENGINE")
    os.environ["GEMMGUARD_ENGINE"] = name or old or "exact"
    try:
        yield
    finally:
        if old is None:
            os.environ.pop("GEMMGUARD_ENGINE", None)
        else:
            os.environ["GEMMGUARD_ENGINE"] = old


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        cfg = WorkbenchConfig.from_file(args.config)
        if args.seed is not None:  # the override is part of the hashed config
            cfg.campaign["seed"] = cfg.raw["campaign"]["seed"] = args.seed
        workers = args.workers if args.workers is not None else int(os.environ.get("GEMMGUARD_WORKERS", "1"))
        with _engine(args.engine):
            STAGE_FNS[args.stage](cfg, Artifacts(cfg, args.out), workers)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    except StageError as exc:
        print(f"stage error: {exc}", file=sys.stderr)
        return 3
    except (WorkbenchError, ValueError, ArithmeticError) as exc:
        print(f"runtime error: {exc}", file=sys.stderr)
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
