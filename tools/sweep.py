"""Threshold (or other knob) sweep of B200 backends through the reference's own
experiment harness: ``stepspec.bench.run_sweep`` drives the
backends exactly as it drives its HTTP / simulated ones and writes
``results.csv``, ``summary.json``, ``traces/*.jsonl`` and the plot data in the
reference schema (``bench.py:25-39``, ``bench.py:366-407``).  The backends'
B200-measured ``BackendProfile`` (the reference's ``profile`` verb,
``cli.py:399-442``) is written next to them as ``profiles.json``.

    python tools/sweep.py --pair 1.5b+7b --knob Threshold --values 3,5,7,9,10 \\
        --schemes SpecReason,BaseOnly --tasks 2 --length 4 --budget 512 --out gpurun_out/sweep

``run_with`` takes any (small, base) pair; ``tests/test_sweep.py`` hands it the
CPU oracle backends to check the harness wiring without a GPU.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def import_reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "stepspec" / "__init__.py").exists():
            sys.path.insert(0, str(p))
            break
    import stepspec

    return stepspec


def parse(argv=None) -> argparse.Namespace:
    ap = argparse.ArgumentParser()
    ap.add_argument("--pair", default="tiny")
    ap.add_argument("--knob", default="Threshold")
    ap.add_argument("--values", default="3,5,7,9,10")
    ap.add_argument("--schemes", default="SpecReason,BaseOnly")
    ap.add_argument("--tasks", type=int, default=2)
    ap.add_argument("--length", type=int, default=4)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--budget", type=int, default=256)
    ap.add_argument("--max-step-tokens", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/sweep")
    ap.add_argument("--no-profile", action="store_true")
    return ap.parse_args(argv)


def run_with(a: argparse.Namespace, small, base) -> dict:
    """Calibrate both backends' profiles, then run the reference sweep."""
    from stepspec.bench import Knob, SweepSpec, run_sweep
    from stepspec.core import AcceptanceThreshold, EngineConfig, Scheme
    from stepspec.simlab import make_tasks

    from paper_2504_07891_b200.profile import measure_profile, profile_dict

    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    profiles = {}
    if not a.no_profile:
        for b in (small, base):
            b.profile = measure_profile(b)
            profiles[b.profile.name] = profile_dict(b.profile)
        (out / "profiles.json").write_text(json.dumps(profiles, indent=2) + "\n")

    knob = Knob(a.knob)
    values = tuple(int(v) for v in a.values.split(","))
    cfg = EngineConfig(threshold=AcceptanceThreshold(7), temperature=0.0, token_budget=a.budget,
                       max_step_tokens=a.max_step_tokens)
    spec = SweepSpec(knob=knob, values=values, base_config=cfg, repeats=a.repeats)
    schemes = tuple(Scheme(s) for s in a.schemes.split(","))
    tasks = make_tasks(a.tasks, a.length, seed=0)
    t0 = time.monotonic()
    res = run_sweep(spec, tasks, small, base, schemes=schemes, output_dir=out)
    summary = {"pair": a.pair, "wall_s": round(time.monotonic() - t0, 2), "cells": len(res.cells),
               "records": len(res.records), "profiles": profiles, "out": str(out)}
    print(json.dumps(summary), flush=True)
    return summary


def main(argv=None) -> dict:
    a = parse(argv)
    stepspec = import_reference()
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.host import reference_types

    small, base = build_pair(a.pair, types=reference_types(stepspec), max_ctx=a.budget + 1024)
    return run_with(a, small, base)


if __name__ == "__main__":
    main()
