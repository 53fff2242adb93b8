"""Run the workbench CLI's seven stages for every golden config and print which artifacts
differ from the reference's (tests/golden/cli), with the first differing lines."""
import difflib
import sys
import tempfile
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200.cli import STAGES, main  # noqa: E402

GOLDEN = Path(__file__).resolve().parents[1] / "tests" / "golden" / "cli"
warnings.simplefilter("ignore", RuntimeWarning)
for d in sorted(GOLDEN.iterdir()):
    with tempfile.TemporaryDirectory() as tmp:
        for stage in STAGES:
            rc = main([stage, "--config", str(d / "config.json"), "--out", tmp])
            if rc:
                print(d.name, stage, "exit", rc)
                break
        for g in sorted(d.iterdir()):
            if g.name == "config.json":
                continue
            o = Path(tmp) / g.name
            if not o.exists():
                print(d.name, g.name, "MISSING")
            elif o.read_bytes() != g.read_bytes():
                diff = list(difflib.unified_diff(g.read_text().splitlines(), o.read_text().splitlines(), lineterm="", n=0))
                print(d.name, g.name, "DIFFERS", len(diff), "diff lines")
                print("\n".join(diff[:int(__import__("os").environ.get("DIFF_LINES", "12"))]))
            else:
                print(d.name, g.name, "ok")
