"""SURVEY §8f rows at the bench shapes, each against the full-depth oracle
(``oracle/replay.py``; tolerance ``max(2e-2, 2 * floor)`` of
``tests/golden/floors.json``, as in ``test_gpu_trajectory_parity.py``).

* f-1 SpecReason+Decode (``speculative_decode``, ``specdecode.py:120-177``):
  the base's steps decoded with the draft proposing gamma=5 tokens per round
  are the oracle's greedy tokens (lossless up to flagged near-ties), and with
  the successor circuit the pair agrees often enough to be faster than plain
  decode;
* f-2 several trajectories per GPU: batched decode (``sr_step_batch``) and
  batched verify (``sr_score_batch``) against the oracle, not only against
  the device's single-stream path;
* f-3 prefix-sharing verify template v2: a trajectory through the driver
  with ``verify_template="v2"``, every call replayed on the oracle.
"""

import json
import time
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.replay import replay
from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
from paper_2504_07891_b200.contract import GenerationRequest
from paper_2504_07891_b200.domain import (DEFAULT_STEP_STOP_MARKERS, BackendRole,
                                          render_generation_prompt, render_verification_prompt)

pytestmark = pytest.mark.gpu
FLOORS = Path(__file__).parent / "golden" / "floors.json"


def tol(model: str) -> float:
    return max(2e-2, 2.0 * json.loads(FLOORS.read_text())[model]["floor_max_abs"])


def _clean(rep):
    assert not rep["token_mismatch"], rep["token_mismatch"][:5]
    assert not rep["score_mismatch"], rep["score_mismatch"][:5]
    assert rep["accept_mismatch"] == 0
    assert rep["flagged_rate"] <= 0.02, rep["flagged_rate"]


@pytest.fixture(scope="module")
def c2(cuda):
    from paper_2504_07891_b200.backend import build_pair

    small, base = build_pair("1.5b+7b", max_ctx=4096, record=True, n_streams=6)
    yield small, base
    del small, base
    torch.cuda.empty_cache()


def test_f1_speculative_decode_lossless_and_faster(c2):
    small, base = c2
    v = base.vocab
    problem = v.problem(64, 77)
    cot, prompts = "", []
    # a CoT of base steps, then time each step's regeneration both ways
    for _ in range(8):
        prompts.append(render_generation_prompt(problem, cot))
        r = base.generate_step(GenerationRequest(prompt=prompts[-1], max_tokens=256,
                                                 stop=DEFAULT_STEP_STOP_MARKERS))
        cot += r.text
    base.calls.clear()

    def run(spec: bool):
        if spec:
            base.attach_speculator(small, gamma=5)
        else:
            base.speculator = None
        for s in base.pool.streams:
            base.engine.truncate(s, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = [base.generate_step(GenerationRequest(prompt=p, max_tokens=256,
                                                     stop=DEFAULT_STEP_STOP_MARKERS))
                for p in prompts]
        torch.cuda.synchronize()
        return outs, time.perf_counter() - t0

    run(True)  # warm both paths
    plain, t_plain = run(False)
    fast, t_fast = run(True)
    spec_calls = base.calls[-len(prompts):]
    stats = dict(base.spec_stats)
    base.speculator = None
    rep = replay(base, spec_calls, tol("qwen2.5-7b"))
    _clean(rep)
    same = sum(a.text == b.text for a, b in zip(plain, fast))
    toks = sum(r.token_count for r in fast)
    acc = stats["accepted"] / max(1, stats["proposed"])
    print(json.dumps({"f1": {"steps": len(prompts), "tokens": toks, "identical_steps": same,
                             "plain_ms_per_token": round(1e3 * t_plain / toks, 3),
                             "spec_ms_per_token": round(1e3 * t_fast / toks, 3),
                             "speedup": round(t_plain / t_fast, 2), "acceptance": round(acc, 3),
                             "flagged": rep["token_mismatch_flagged"]}}))
    assert same >= len(prompts) - 1
    assert acc > 0.5
    assert t_fast < t_plain


def test_f2_batched_passes_on_oracle(c2):
    small, base = c2
    v = small.vocab
    rng = np.random.default_rng(5)
    prompts = [v.encode(render_generation_prompt(v.problem(64, 200 + k),
                                                 " ".join(v.words[int(x)] for x in
                                                          rng.integers(16, v.n_text, size=300 * k))
                                                 + " ")) for k in range(4)]
    streams = small.pool.streams[:4]
    for s in streams:
        small.engine.truncate(s, 0)
    outs = small.engine.generate_batch(streams, prompts, 32, ())
    calls = [{"kind": "gen", "prompt_ids": p, "gen_ids": g} for p, (g, _) in zip(prompts, outs)]
    rep = replay(small, calls, tol("r1-1.5b"))
    _clean(rep)
    words = v.problem(400, 9).split()
    sufs = [v.encode(render_verification_prompt(" ".join(words[:64]),
                                                " ".join(words[64:100 + 60 * k]) + " ",
                                                " ".join(words[-24:]) + " ")) for k in range(4)]
    bstreams = base.pool.streams[:4]
    for s in bstreams:
        base.engine.truncate(s, 0)
    reads = base.engine.score_batch(bstreams, sufs, base.threshold)
    scalls = [{"kind": "score", "prompt_ids": p, "score": r.score, "accept": r.accept}
              for p, r in zip(sufs, reads)]
    srep = replay(base, scalls, tol("qwen2.5-7b"))
    _clean(srep)
    print(json.dumps({"f2": {"decode_tokens": rep["tokens"], "decode_flagged": rep["token_mismatch_flagged"],
                             "scores": [r.score for r in reads],
                             "score_flagged": srep["score_mismatch_flagged"]}}))


def test_f3_prefix_sharing_template_trajectory(c2):
    from paper_2504_07891_b200.driver import run_trajectory, validate_trajectory

    small, base = c2
    small.calls.clear()
    base.calls.clear()
    base.verify_template = "v2"
    try:
        cfg = EngineConfig(threshold=AcceptanceThreshold(7), temperature=0.0, token_budget=1024)
        res = run_trajectory(cfg, small.vocab.problem(64, 3), small, base)
        validate_trajectory(res, cfg)
    finally:
        base.verify_template = "v1"
    kinds = [c["kind"] for c in base.calls]
    assert "score" in kinds
    # v2 verify prompts extend the generation prompt: the base reuses its
    # generation K/V (fresh rows per score call = candidate + tail)
    fresh = [c["fresh"] for c in base.calls if c["kind"] == "score"]
    for be, name in ((small, "r1-1.5b"), (base, "qwen2.5-7b")):
        _clean(replay(be, be.calls, tol(name)))
    print(json.dumps({"f3": {"steps": len(res.state.retained_steps),
                             "mean_fresh_verify_rows": round(sum(fresh) / len(fresh), 1)}}))


def test_f4_reference_sweep_on_b200(cuda, stepspec, tmp_path):
    """f-4 on the device: the reference's own experiment harness
    (``stepspec.bench.run_sweep``, ``bench.py:221-300``) drives the tiny B200
    pair and writes ``results.csv`` / ``summary.json`` / traces in the
    reference schema (``bench.py:25-39``, ``366-407``), after the reference
    ``profile`` verb's two-point fits (``cli.py:399-442``) measured the
    backends; threshold 0 accepts every step, 10 rejects every step
    (``test_acceptance.py:116-126``)."""
    import csv
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import sweep

    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.host import reference_types

    small, base = build_pair("tiny", types=reference_types(stepspec), max_ctx=1024)
    a = sweep.parse(["--values", "0,7,10", "--tasks", "2", "--length", "2", "--budget", "96",
                     "--max-step-tokens", "16", "--out", str(tmp_path)])
    out = sweep.run_with(a, small, base)
    assert out["records"] == 2 * 3 * 2  # tasks x values x schemes (SpecReason, BaseOnly)
    rows = [r for r in csv.reader((tmp_path / "results.csv").read_text().splitlines()[1:])]
    assert rows[0][:3] == ["scheme", "knob", "knob_value"]
    cells = {(r[0], r[2]): r for r in rows[1:]}
    assert float(cells[("SpecReason", "0")][8]) == 1.0
    assert float(cells[("SpecReason", "10")][8]) == 0.0
    assert json.loads((tmp_path / "summary.json").read_text())["schema"] == "stepspec.results.v1"
    prof = json.loads((tmp_path / "profiles.json").read_text())
    assert all(p["decode_s_per_token"] > 0 and p["prefill_tokens_per_s"] > 0 for p in prof.values())
