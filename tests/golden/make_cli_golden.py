"""Golden artifacts of the workbench CLI and the protection planner, written by the REFERENCE.

Imports the unmodified reference package from /root/reference/pkg/src (this
container only) and records:

  cli/<name>/config.json   a workbench config (output_dir is the fixed string "out";
                           artifacts were written through --out, which is not hashed)
  cli/<name>/*             every artifact of the seven stages run in order
  planning.json            analysis.select_layers (greedy and exact, with cost / memory
                           totals) and analysis.build_coverage_curve on seeded vectors

Run:  python tests/golden/make_cli_golden.py      (writes next to this file)
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from gemmguard import analysis as A  # noqa: E402
from gemmguard.cli import STAGES, main  # noqa: E402

HERE = Path(__file__).resolve().parent

CONFIGS = {
    # the reference's own CLI test config (tests/test_cli.py:9-22)
    "fp16_toy": {
        "model": {"blocks": 1, "dim": 8, "tokens": 4, "classes": 5, "seed": 17, "dtype": "binary16-emulated"},
        "dataset": {"size": 40, "seed": 3},
        "campaign": {"n_per_layer": 8, "seed": 7},
        "guard": {"confidence": 0.999, "precision": "binary64", "target_coverage": 0.9, "per_sample": True},
        "correction": {"kind": "replay", "max_replays": 3},
        "output_dir": "out",
    },
    # an int8 toy through the automatic precision choice (int64 checks) and two fault modes
    "int8_toy": {
        "model": {"blocks": 2, "dim": 16, "tokens": 6, "classes": 7, "seed": 5, "dtype": "int8"},
        "dataset": {"size": 48, "seed": 11},
        "campaign": {"n_per_layer": 12, "seed": 21},
        "guard": {"confidence": 0.9999, "precision": "auto", "target_coverage": 0.95},
        "output_dir": "out",
    },
    # binary32 with the automatic precision choice and the batch-mean statistic
    "fp32_toy": {
        "model": {"blocks": 1, "dim": 12, "tokens": 5, "classes": 4, "seed": 9, "dtype": "binary32"},
        "dataset": {"size": 32, "seed": 4},
        "campaign": {"n_per_layer": 6, "seed": 13},
        "guard": {"confidence": 0.999, "precision": "auto", "target_coverage": 0.8, "per_sample": False},
        "output_dir": "out",
    },
}


def cli_goldens() -> None:
    root = HERE / "cli"
    if root.exists():
        shutil.rmtree(root)
    for name, cfg in CONFIGS.items():
        dst = root / name
        dst.mkdir(parents=True)
        (dst / "config.json").write_text(json.dumps(cfg, indent=2) + "\n")
        with tempfile.TemporaryDirectory() as tmp:
            for stage in STAGES:
                code = main([stage, "--config", str(dst / "config.json"), "--out", tmp])
                if code != 0:
                    raise SystemExit(f"{name}: reference stage {stage} exited {code}")
            for p in sorted(Path(tmp).iterdir()):
                shutil.copy(p, dst / p.name)
        print(name, sorted(p.name for p in dst.iterdir()))


def planning_golden() -> None:
    rng = np.random.default_rng(2310)
    cases = []
    for t in range(60):
        n = int(rng.integers(2, 13))
        v = rng.random(n) * (rng.random(n) < 0.8)
        if v.sum() == 0:
            v[int(rng.integers(0, n))] = 0.5
        c = rng.random(n) + (0.0 if t % 7 == 0 else 0.01)
        if t % 5 == 0:
            c[int(rng.integers(0, n))] = 0.0  # zero-cost layers rank first
        mem = rng.random(n)
        head = n - 1 if t % 3 else None
        target = float([0.3, 0.8, 0.95, 1.0][t % 4])
        case = {"v": v.tolist(), "c": c.tolist(), "mem": mem.tolist(), "head": head, "target": target,
                "total_compute": float(c.sum() * 3.0), "total_memory": float(mem.sum() * 2.0)}
        for method in ("greedy", "exact"):
            try:
                plan = A.select_layers(v, c, target, head_index=head, method=method,
                                       total_compute=case["total_compute"], memory_costs=mem,
                                       total_memory=case["total_memory"])
                case[method] = plan.to_json()
            except ValueError as exc:
                case[method] = {"error": str(exc)}
        case["curve"] = A.build_coverage_curve(v, c).to_csv()
        cases.append(case)
    (HERE / "planning.json").write_text(json.dumps(cases, indent=1) + "\n")
    print("planning cases", len(cases))


if __name__ == "__main__":
    cli_goldens()
    planning_golden()
