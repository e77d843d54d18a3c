"""The reference arm the driver runs (``bench.py --impl reference``) works on
the committed trace (``bench_data/``): the unmodified reference engine
replays the recorded windows and prices their calls on the host cores.  A
short run (one timed step per window) checks the trace format, the replay
backends and the per-window step accounting without a GPU."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_on_committed_trace(stepspec):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "4", "--warmup", "3", "--ref-layer-frac", "0.05",
                          "--ref-decode-cap", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "unavailable" not in line, line
    assert line["impl"] == "reference" and line["steps"] == 4 and line["value"] > 0
    assert line["loop"]["tokens"] > 0
    assert line["config"]["pair"] == "1.5b+32b"
