"""Full-depth trajectory parity at the bench shapes (the north-star target).

The *unmodified reference engine* (``stepspec.engine.run_trajectory``,
``engine.py:297-354``, installed in ``baseline/_ref``) drives the two
``B200Backend``s of a model pair for a whole trajectory -- C3: R1-1.5B-shape
draft + QwQ-32B-shape base, threshold 7, 8192-token thinking budget; C2:
1.5B + 7B, 4096 -- and ``validate_trajectory`` (``engine.py:715-754``)
accepts the result.  Then every backend call of the trajectory (every draft
and fallback token, every verify readout, the answer) is replayed through
the full-depth, layer-streamed fp32 oracle (``oracle/replay.py``) by teacher
forcing:

* a device token must equal the oracle's argmax unless the oracle's gap to
  it is below the logit tolerance (flagged near-tie);
* a device judge score / accept bit must equal the oracle's ``extract_score``
  readout unless the readout's deciding gap is below the tolerance (flagged);
* the device's reported top-2 margins, and the prefill path's fp32 logits of
  the longest context, must match the oracle within the tolerance.

Tolerance (per model, stated): ``max(2e-2, 2 * floor)``, ``floor`` being the
oracle's own fp32-vs-fp64 max-abs logit difference at that shape and full
depth on identical bf16 storage points (``tests/golden/floors.json``,
measured by ``tools/measure_floors.py``) -- how far two exact fp32
implementations of the same bf16-storage model are apart.  It is not derived
from the device's error.
"""

import json
import os
from pathlib import Path

import pytest
import torch

from oracle.replay import replay
from paper_2504_07891_b200.host import reference_types

pytestmark = pytest.mark.gpu

FLOORS_PATH = Path(__file__).parent / "golden" / "floors.json"


def tolerance(model: str) -> float:
    floors = json.loads(FLOORS_PATH.read_text())
    return max(2e-2, 2.0 * floors[model]["floor_max_abs"])


CASES = {
    # pair, budget, problem seed, max flagged fraction
    "C3": ("1.5b+32b", int(os.environ.get("SR_C3_BUDGET", "8192")), 0),
    "C2": ("1.5b+7b", int(os.environ.get("SR_C2_BUDGET", "4096")), 1),
}


@pytest.mark.parametrize("case", ["C3", "C2"])
def test_full_depth_trajectory_replays_on_oracle(cuda, stepspec, case):
    from stepspec import engine as reng
    from stepspec.core import AcceptanceThreshold, EngineConfig

    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.shapes import PAIRS

    pair, budget, seed = CASES[case]
    T = reference_types(stepspec)
    small, base = build_pair(pair, max_ctx=budget + 512, types=T, record=True)
    cfg = EngineConfig(threshold=AcceptanceThreshold(7), temperature=0.0, token_budget=budget)
    res = reng.run_trajectory(cfg, small.vocab.problem(64, seed), small, base)
    reng.validate_trajectory(res, cfg)
    kept = res.state.retained_steps
    n_spec = sum(1 for s in kept if s.producer.value == "Speculator")
    summary = {"case": case, "pair": pair, "budget": budget, "steps": len(kept),
               "accepted": n_spec, "rejected": len(res.rejected_steps),
               "thinking_tokens": res.state.thinking_tokens_used}
    reports = {}
    for be, name in ((small, PAIRS[pair][0]), (base, PAIRS[pair][1])):
        tol = tolerance(name)
        rep = replay(be, be.calls, tol, logits_check=64)
        reports[name] = rep
        assert not rep["token_mismatch"], (name, rep["token_mismatch"][:5])
        assert not rep["score_mismatch"], (name, rep["score_mismatch"][:5])
        assert rep["accept_mismatch"] == 0, name
        assert rep["margin_err_max"] <= tol, (name, rep["margin_err_max"], tol)
        assert rep["logits_max_abs"] <= tol, (name, rep["logits_max_abs"], tol)
        # near-ties are rare: a broken kernel would flag far more
        assert rep["flagged_rate"] <= 0.02, (name, rep["flagged_rate"])
    summary["replay"] = reports
    print(json.dumps(summary))
    out = os.environ.get("SR_PARITY_REPORT")
    if out:
        p = Path(out)
        p.parent.mkdir(parents=True, exist_ok=True)
        with p.open("a") as f:
            f.write(json.dumps(summary) + "\n")
    assert len(kept) >= 40 and max(len(c["prompt_ids"]) for c in base.calls) >= 4096
    del small, base
    torch.cuda.empty_cache()
