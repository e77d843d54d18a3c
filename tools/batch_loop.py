"""Same SpecReason trajectories, serial vs concurrent with batched device
passes: B problems x S steps each, on one GPU.  Prints wall
time, CoT tokens/s and whether every trajectory matched its serial twin.

    python tools/batch_loop.py --pair 1.5b+7b --b 8 --steps 12
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--pair", default="1.5b+7b")
    ap.add_argument("--b", type=int, default=8)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--threshold", type=int, default=7)
    ap.add_argument("--budget", type=int, default=4096)
    ap.add_argument("--max-step-tokens", type=int, default=256)
    a = ap.parse_args()
    from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.batching import BatchScheduler
    from paper_2504_07891_b200.driver import SpecReasonSession
    from paper_2504_07891_b200.shapes import PAIRS, get_spec
    from paper_2504_07891_b200.vocab import shared_vocab

    small, base = build_pair(a.pair, max_ctx=a.budget + 512, threshold=a.threshold,
                             n_streams=2 * a.b + 2, max_tokens=1024)
    vocab = shared_vocab(get_spec(PAIRS[a.pair][0]).vocab_text)
    cfg = EngineConfig(threshold=AcceptanceThreshold(a.threshold), temperature=0.0,
                       token_budget=a.budget, max_step_tokens=a.max_step_tokens)
    problems = [vocab.problem(64, 500 + k) for k in range(a.b)]

    def trajectory(s, b, prob):
        sess = SpecReasonSession(cfg, prob, s, b)
        out = []
        for _ in range(a.steps):
            o = sess.step()
            if o is None:
                break
            out.append((o.step.text, o.step.producer.value, o.step.accepted))
        return out

    trajectory(small, base, problems[0])  # warm-up
    torch.cuda.synchronize()
    s0 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
    t0 = time.perf_counter()
    serial = [trajectory(small, base, p) for p in problems]
    torch.cuda.synchronize()
    t_serial = time.perf_counter() - t0
    ds, db = small.engine.stats.minus(s0[0]), base.engine.stats.minus(s0[1])
    dev = {"small_decode_ms": round(ds.decode_ms), "small_decode_tokens": ds.decode_tokens,
           "small_prefill_ms": round(ds.prefill_ms), "small_prefill_tokens": ds.prefill_tokens,
           "base_prefill_ms": round(db.prefill_ms), "base_prefill_tokens": db.prefill_tokens,
           "base_decode_ms": round(db.decode_ms), "calls": ds.calls + db.calls}
    s1 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
    sched = BatchScheduler(small, base)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batched = sched.run([lambda s, b, p=p: trajectory(s, b, p) for p in problems])
    torch.cuda.synchronize()
    t_batched = time.perf_counter() - t0
    sched.close()
    ds, db = small.engine.stats.minus(s1[0]), base.engine.stats.minus(s1[1])
    devb = {"small_ms": round(ds.decode_ms + ds.prefill_ms), "base_ms": round(db.decode_ms + db.prefill_ms),
            "calls": ds.calls + db.calls}
    tokens = sum(len(t.split()) for traj in serial for t, _, _ in traj)
    same = sum(1 for x, y in zip(serial, batched) if x == y)
    acc = sum(1 for traj in serial for _, _, ok in traj if ok) / max(1, sum(len(t) for t in serial))
    print(json.dumps({"pair": a.pair, "B": a.b, "steps_per_trajectory": a.steps, "cot_tokens": tokens,
                      "accepted_fraction": round(acc, 3),
                      "serial_s": round(t_serial, 2), "batched_s": round(t_batched, 2),
                      "serial_tok_s": round(tokens / t_serial, 1),
                      "batched_tok_s": round(tokens / t_batched, 1),
                      "speedup": round(t_serial / t_batched, 2),
                      "trajectories_identical": f"{same}/{a.b}",
                      "mean_pass_size": round(sum(sched.batches) / len(sched.batches), 2),
                      "serial_device": dev, "batched_device": devb}), flush=True)


if __name__ == "__main__":
    main()
