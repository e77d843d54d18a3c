"""The reference's experiment harness (``stepspec.bench.run_sweep``) driving
this package's backend interface, and the reference ``profile`` verb's
two-point fits (``cli.py:399-442``) through ``generate_step``.
CPU: the oracle backends stand in for the B200 ones."""

import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))


def test_reference_sweep_writes_reference_schema(stepspec, tmp_path):
    import sweep
    from oracle.ref_engine import oracle_backend
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.host import reference_types

    T = reference_types(stepspec)
    small = oracle_backend("tiny-draft", BackendRole.SMALL, types=T)
    base = oracle_backend("tiny-base", BackendRole.BASE, types=T)
    a = sweep.parse(["--values", "0,10", "--tasks", "1", "--length", "2", "--budget", "64",
                     "--max-step-tokens", "16", "--out", str(tmp_path)])
    out = sweep.run_with(a, small, base)
    assert out["records"] == 4
    rows = [r for r in csv.reader((tmp_path / "results.csv").read_text().splitlines()[1:])]
    assert rows[0][:3] == ["scheme", "knob", "knob_value"]
    cells = {(r[0], r[2]): r for r in rows[1:]}
    # threshold 0 accepts every step; threshold 10 rejects every step (test_acceptance.py:116-126)
    assert float(cells[("SpecReason", "0")][8]) == 1.0
    assert float(cells[("SpecReason", "10")][8]) == 0.0
    summary = json.loads((tmp_path / "summary.json").read_text())
    assert summary["schema"] == "stepspec.results.v1"
    assert (tmp_path / "traces" / "SpecReason_0.jsonl").exists()
    prof = json.loads((tmp_path / "profiles.json").read_text())
    for p in prof.values():
        assert p["decode_s_per_token"] > 0 and p["prefill_tokens_per_s"] > 0
