"""Per-path timing of one model: prefill a context, then greedy-decode.

    python tools/decode_profile.py qwen2.5-7b --ctx 2048 --new 32 [--reps 3]

Prints CUDA-event times of the prefill and the decode graph (per token) and
the achieved HBM GB/s of decode against the algorithmic bytes.
Small enough to run under ncu for a per-kernel launch list."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--new", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--verify", type=int, default=80, help="verify-prefill tokens (base models)")
    a = ap.parse_args()
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.shapes import get_spec

    spec = get_spec(a.model)
    b = B200Backend(spec, BackendRole.BASE, max_ctx=a.ctx + a.new + a.verify + 64)
    eng = b.engine
    g = torch.Generator().manual_seed(0)
    ctx = torch.randint(16, spec.vocab_text, (a.ctx,), generator=g).tolist()
    s = b.pool.streams[0]
    out = {"model": a.model, "ctx": a.ctx}
    for rep in range(a.reps):
        eng.truncate(s, 0)
        no_stop = ()
        gen, _ = eng.generate(s, ctx, a.new, no_stop)
        t = eng.model.timing()
        n = len(gen) - 1
        per_tok = t.decode_ms / max(1, n)
        byts = sum(spec.decode_bytes(a.ctx + i) for i in range(n)) / max(1, n)
        out[f"rep{rep}"] = {"prefill_ms": round(t.prefill_ms, 3),
                            "prefill_tok_per_s": round(a.ctx / (t.prefill_ms * 1e-3)),
                            "decode_ms_per_token": round(per_tok, 4),
                            "decode_GBps": round(byts / (per_tok * 1e-3) / 1e9, 1)}
        # verify-sized prefill on top of the context
        ids = torch.randint(16, spec.vocab_text, (a.verify,), generator=g).tolist()
        keep = len(s.ids)
        eng.forward_logits(s, ids, all_rows=False)
        eng.truncate(s, keep)
        torch.cuda.synchronize()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
