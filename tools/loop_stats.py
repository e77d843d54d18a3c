"""SpecReason loop statistics vs weight-circuit settings (calibration tool).

Runs the driver's ``SpecReasonSession`` over several problems for each
combination of draft / base ``ModelSpec`` overrides (e.g. the successor
circuit's ``succ_gain``, ``embed_std``, the judge's ``cue_gain``) and prints:
the fraction of generated tokens that follow the successor circuit, draft /
base generation lengths (mean, median, p90, capped at 256), accepted
fraction, retained tokens per step, score histogram and the device CoT
tokens/s.

    python tools/loop_stats.py --pair 1.5b+7b --draft-over "embed_std=1,succ_gain=0.8" \
        --base-over "embed_std=1,succ_gain=0.8|embed_std=1,succ_gain=1.2"
"""

from __future__ import annotations

import argparse
import collections
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig  # noqa: E402
from paper_2504_07891_b200.backend import B200Backend  # noqa: E402
from paper_2504_07891_b200.domain import BackendRole  # noqa: E402
from paper_2504_07891_b200.driver import SpecReasonSession  # noqa: E402
from paper_2504_07891_b200.shapes import PAIRS, get_spec, successor_perm  # noqa: E402


def overrides(text: str) -> list[dict]:
    """'a=1,b=2|a=3' -> [{'a': 1.0, 'b': 2.0}, {'a': 3.0}] ('-' = defaults)."""
    out = []
    for part in text.split("|"):
        d = {}
        for kv in filter(None, part.split(",")):
            if kv == "-":
                continue
            k, v = kv.split("=")
            d[k] = tuple(float(x) for x in v.split(":")) if ":" in v else float(v)
        out.append(d)
    return out


def follow_rate(calls, succ) -> float:
    """Fraction of generated tokens that are the successor-circuit choice."""
    hit = tot = 0
    for c in calls:
        if c["kind"] != "gen":
            continue
        prev = c["prompt_ids"][-1]
        for t in c["gen_ids"]:
            hit += int(succ[prev]) == t
            tot += 1
            prev = t
    return round(hit / max(1, tot), 3)


def stats(xs):
    if not xs:
        return {}
    xs = sorted(xs)
    return {"mean": round(statistics.mean(xs), 1), "median": statistics.median(xs),
            "p90": xs[int(0.9 * len(xs))], "capped": round(sum(x >= 256 for x in xs) / len(xs), 3),
            "n": len(xs)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--pair", default="1.5b+7b")
    ap.add_argument("--draft-over", default="-", help="spec overrides, '|'-separated sets")
    ap.add_argument("--base-over", default="-")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--problems", type=int, default=3)
    ap.add_argument("--threshold", type=int, default=7)
    ap.add_argument("--budget", type=int, default=8192)
    args = ap.parse_args()
    cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                       token_budget=args.budget)
    dn, bn = PAIRS[args.pair]
    for od in overrides(args.draft_over):
        for ob in overrides(args.base_over):
            small = base = None
            torch.cuda.empty_cache()
            small = B200Backend(get_spec(dn, **od), BackendRole.SMALL, max_ctx=args.budget + 512,
                                record=True)
            base = B200Backend(get_spec(bn, **ob), BackendRole.BASE, max_ctx=args.budget + 512,
                               record=True, threshold=args.threshold)
            succ = successor_perm(small.vocab.n_text)[0]
            small.calls.clear()
            base.calls.clear()
            s0 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
            outs = []
            t0 = time.time()
            for p in range(args.problems):
                sess = SpecReasonSession(cfg, small.vocab.problem(64, p), small, base)
                for _ in range(args.steps):
                    o = sess.step()
                    if o is None:
                        break
                    outs.append(o)
            ds = small.engine.stats.minus(s0[0])
            db = base.engine.stats.minus(s0[1])
            dev_ms = ds.prefill_ms + ds.decode_ms + db.prefill_ms + db.decode_ms
            toks = sum(o.step.token_count for o in outs)
            scores = collections.Counter(c["score"] for c in base.calls if c["kind"] == "score")
            print(json.dumps({
                "draft": od, "base": ob,
                "follow": [follow_rate(small.calls, succ), follow_rate(base.calls, succ)],
                "draft_len": stats([len(c["gen_ids"]) for c in small.calls]),
                "base_len": stats([len(c["gen_ids"]) for c in base.calls if c["kind"] == "gen"]),
                "retained": stats([o.step.token_count for o in outs]),
                "accepted": round(sum(o.action.value == "AcceptedSpeculation" for o in outs)
                                  / max(1, len(outs)), 3),
                "scores": dict(sorted(scores.items())),
                "cot_tok_s_device": round(toks / (dev_ms * 1e-3), 1) if dev_ms else None,
                "ms_per_step": round(dev_ms / max(1, len(outs)), 1),
                "wall_s": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
