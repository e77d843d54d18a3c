"""Bring-up probe (run under gpurun): exercise every C-ABI entry point on the
tiny pair against the CPU oracle and time 1.5B / 7B decode.  Prints JSON-ish
lines; failures are reported per stage so one call yields maximal signal."""

from __future__ import annotations

import json
import sys
import time
import traceback
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402


def stage(name):
    def deco(fn):
        def run(*a, **k):
            t0 = time.time()
            try:
                out = fn(*a, **k)
                print(json.dumps({"stage": name, "ok": True, "s": round(time.time() - t0, 2),
                                  **(out or {})}), flush=True)
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"stage": name, "ok": False, "err": repr(exc)[:500]}), flush=True)
                traceback.print_exc()
        return run
    return deco


@stage("tiny-logits")
def tiny_logits():
    from oracle.ref_engine import RefEngine
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
    from paper_2504_07891_b200.shapes import get_spec, make_weights
    from paper_2504_07891_b200.vocab import shared_vocab
    out = {}
    for name in ("tiny-draft", "tiny-base"):
        spec = get_spec(name)
        vocab = shared_vocab(spec.vocab_text)
        w = make_weights(spec, 0)
        gpu = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=2048)
        ref = RefEngine(spec, w, vocab)
        ids = vocab.encode(render_generation_prompt(vocab.problem(64, 1), "")) * 5  # 330 tokens
        s = gpu.pool.streams[0]
        got = gpu.engine.forward_logits(s, ids).cpu()
        want = ref.logits_teacher_forced(ids)
        V = spec.vocab_text
        err = (got[:, :V] - want[:, :V]).abs().max().item()
        agree = (got[:, :V].argmax(-1) == want[:, :V].argmax(-1)).float().mean().item()
        # incremental: prefill in two pieces, last-row logits
        s2 = gpu.pool.streams[1]
        gpu.engine.forward_logits(s2, ids[:100], all_rows=False)
        inc = gpu.engine.forward_logits(s2, ids[100:], all_rows=True).cpu()
        err_inc = (inc[:, :V] - want[100:, :V]).abs().max().item()
        out[name] = {"maxabs": err, "argmax_agree": agree, "maxabs_incremental": err_inc}
    return out


@stage("tiny-trajectory")
def tiny_trajectory():
    from oracle.ref_engine import oracle_backend
    from paper_2504_07891_b200 import (AcceptanceThreshold, EngineConfig, run_trajectory,
                                       validate_trajectory)
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.driver import trace_signature
    from paper_2504_07891_b200.vocab import shared_vocab
    small, base = build_pair("tiny", max_ctx=2048, record=True)
    osmall = oracle_backend("tiny-draft", BackendRole.SMALL)
    obase = oracle_backend("tiny-base", BackendRole.BASE)
    v = shared_vocab(4096)
    cfg = EngineConfig(threshold=AcceptanceThreshold(7), temperature=0.0, max_step_tokens=32,
                       token_budget=256)
    res = {}
    same = 0
    for p in range(6):
        prob = v.problem(64, p)
        t0 = time.time()
        g = run_trajectory(cfg, prob, small, base)
        t1 = time.time()
        validate_trajectory(g, cfg)
        o = run_trajectory(cfg, prob, osmall, obase)
        same += trace_signature(g) == trace_signature(o)
        res[p] = {"steps": len(g.state.retained_steps), "rej": len(g.rejected_steps),
                  "acc": g.metrics.accepted_fraction, "gpu_s": round(t1 - t0, 3),
                  "ms_per_step": round(1000 * sum(s.latency.total_s for s in g.state.retained_steps)
                                       / max(1, len(g.state.retained_steps)), 3)}
    res["identical_to_oracle"] = same
    return res


@stage("decode-timing")
def decode_timing(pair):
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.contract import GenerationRequest, VerificationRequest
    from paper_2504_07891_b200.domain import render_generation_prompt
    from paper_2504_07891_b200.vocab import shared_vocab
    t0 = time.time()
    small, base = build_pair(pair, max_ctx=4096 + 512)
    t_init = time.time() - t0
    v = shared_vocab(small.engine.spec.vocab_text)
    out = {"init_s": round(t_init, 1)}
    for name, b in (("draft", small), ("base", base)):
        prompt = render_generation_prompt(v.problem(64, 3), " ".join(v.words[20:20 + 4000]) + " ")
        req = GenerationRequest(prompt=prompt, max_tokens=64, stop=())
        b.generate_step(req)  # warm (prefill 4K)
        b.generate_step(req)
        eng = b.engine
        tm = eng.model.timing()
        r = b.generate_step(GenerationRequest(prompt=prompt + "kab ", max_tokens=64, stop=()))
        tm = eng.model.timing()
        spec = eng.spec
        ctx = len(b.pool.streams[0].ids)
        n = r.token_count
        dec_ms = tm.decode_ms / max(1, n - 1)
        bytes_tok = spec.decode_bytes(ctx)
        out[name] = {"tokens": n, "prefill_ms": round(tm.prefill_ms, 3),
                     "prefill_tokens": tm.prefill_tokens,
                     "decode_ms_per_tok": round(dec_ms, 4),
                     "decode_GBps": round(bytes_tok / dec_ms / 1e6, 1), "ctx": ctx,
                     "wall_s": r.measured_latency_s}
    # verify timing
    vr = VerificationRequest(problem=v.problem(64, 3), cot_prefix=" ".join(v.words[20:20 + 4000]) + " ",
                             candidate_step=" ".join(v.words[5000:5024]) + " ")
    base.score_step(vr)
    vr2 = VerificationRequest(problem=vr.problem, cot_prefix=vr.cot_prefix + " ".join(v.words[6000:6024]) + " ",
                              candidate_step=" ".join(v.words[7000:7024]) + " ")
    try:
        base.score_step(vr2)
    except Exception:
        pass
    tm = base.engine.model.timing()
    out["verify"] = {"ms": round(tm.prefill_ms, 3), "tokens": tm.prefill_tokens}
    return out


if __name__ == "__main__":
    print(json.dumps({"device": torch.cuda.get_device_name(0)}), flush=True)
    tiny_logits()
    tiny_trajectory()
    for pair in sys.argv[1:]:
        decode_timing(pair)
