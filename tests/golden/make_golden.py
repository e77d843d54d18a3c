"""Generate the committed golden trajectories (run here, where the reference
package is mounted; the GPU box only reads the JSON).

The UNMODIFIED reference engine (``stepspec.engine.run_trajectory`` /
``run_vanilla`` from /root/reference/pkg/src) drives the CPU oracle backends
(bound to the reference's own result types) on configuration C1 of
BASELINE.json: tiny random-init pair, greedy, threshold 7, 64-token prompts,
steps of <= 32 tokens, 256-token thinking budget.  For each trajectory the
fixture stores the timing-free trajectory signature and every backend call
(prompt ids, generated ids, scores) so device runs can be replayed.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import stepspec  # noqa: E402
from stepspec import engine as reng  # noqa: E402
from stepspec.core import AcceptanceThreshold, EngineConfig  # noqa: E402

from oracle.ref_engine import oracle_backend  # noqa: E402
from paper_2504_07891_b200.domain import BackendRole  # noqa: E402
from paper_2504_07891_b200.driver import trace_signature  # noqa: E402
from paper_2504_07891_b200.host import reference_types  # noqa: E402
from paper_2504_07891_b200.vocab import shared_vocab  # noqa: E402

OUT = Path(__file__).with_name("c1_trajectories.json")
C1 = dict(temperature=0.0, max_step_tokens=32, token_budget=256)
PROBLEMS = range(6)


def ids_digest(ids) -> str:
    return hashlib.sha1(",".join(map(str, ids)).encode()).hexdigest()[:16]


def _slim(call: dict) -> dict:
    c = dict(call)
    ids = c.pop("prompt_ids")
    c["prompt_len"], c["prompt_digest"] = len(ids), ids_digest(ids)
    return c


def main() -> None:
    T = reference_types(stepspec)
    vocab = shared_vocab(4096)
    out = {"config": C1, "models": ["tiny-draft", "tiny-base"], "seed": 0, "cases": []}
    for thr in (7, 10, 0):
        for p in PROBLEMS if thr == 7 else range(2):
            small = oracle_backend("tiny-draft", BackendRole.SMALL, types=T, record=True)
            base = oracle_backend("tiny-base", BackendRole.BASE, types=T, record=True,
                                  threshold=thr)
            cfg = EngineConfig(threshold=AcceptanceThreshold(thr), **C1)
            problem = vocab.problem(64, p)
            res = reng.run_trajectory(cfg, problem, small, base)
            reng.validate_trajectory(res, cfg)
            case = {"problem_seed": p, "threshold": thr, "kind": "spec_reason",
                    "signature": trace_signature(res),
                    "small_calls": [_slim(c) for c in small.calls],
                    "base_calls": [_slim(c) for c in base.calls]}
            out["cases"].append(case)
            if thr == 10:
                vb = oracle_backend("tiny-base", BackendRole.BASE, types=T)
                van = reng.run_vanilla(cfg, problem, vb)
                out["cases"].append({"problem_seed": p, "threshold": thr, "kind": "vanilla_base",
                                     "signature": trace_signature(van)})
            print(f"thr={thr} problem={p}: {len(res.state.retained_steps)} steps, "
                  f"{len(res.rejected_steps)} rejected", flush=True)
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
