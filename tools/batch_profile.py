"""Throughput of several trajectories per GPU: B streams on a
C-token context each, then
  * verify: one judge readout per stream for an M-token step, batched
    (``score_batch``, one pass of B*M rows) vs one call per stream;
  * decode: N greedy tokens per stream, batched (``generate_batch``, one
    weight stream per token for all B) vs the persistent single-stream kernel.
Prints one JSON line per (model, B).

    python tools/batch_profile.py qwen2.5-7b --ctx 2048 --m 80 --b 1,2,4,8
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--m", type=int, default=80)
    ap.add_argument("--new", type=int, default=32)
    ap.add_argument("--b", default="1,2,4,8")
    ap.add_argument("--max-tokens", type=int, default=1024)
    a = ap.parse_args()
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.shapes import get_spec

    bs = [int(x) for x in a.b.split(",")]
    nmax = max(bs)
    spec = get_spec(a.model)
    eng = B200Backend(spec, BackendRole.BASE, max_ctx=a.ctx + a.m + a.new + 64,
                      max_tokens=a.max_tokens, n_streams=2 * nmax).engine
    rng = np.random.default_rng(0)
    streams = eng.streams[:nmax]
    ctxs = [[int(x) for x in rng.integers(16, spec.vocab_text, size=a.ctx)] for _ in range(nmax)]
    for st, c in zip(streams, ctxs):
        eng.truncate(st, 0)
        eng.prefill(st, c)

    def sync_time(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    for b in bs:
        sts = streams[:b]
        sufs = [[int(x) for x in rng.integers(16, spec.vocab_text, size=a.m)] for _ in range(b)]
        res = {"model": a.model, "ctx": a.ctx, "B": b, "m": a.m}
        # verify: batched vs one call per stream (rolled back after each timing)
        best_b, best_s = 1e9, 1e9
        for _ in range(3):
            best_b = min(best_b, sync_time(lambda: eng.score_batch(sts, sufs, 7)))
            for st in sts:
                eng.truncate(st, a.ctx)
            best_s = min(best_s, sync_time(lambda: [eng.score(st, sf, 7) for st, sf in zip(sts, sufs)]))
            for st in sts:
                eng.truncate(st, a.ctx)
        res.update(verify_batched_ms=round(best_b * 1e3, 3), verify_serial_ms=round(best_s * 1e3, 3),
                   verify_speedup=round(best_s / best_b, 2))
        # decode: batched steps vs the persistent kernel, stream by stream
        seed = [[int(rng.integers(16, spec.vocab_text))] for _ in range(b)]
        tb = sync_time(lambda: eng.generate_batch(sts, seed, a.new, ()))
        toks_b = sum(len(st.ids) - a.ctx for st in sts)  # fed tokens
        for st in sts:
            eng.truncate(st, a.ctx)
        ts = sync_time(lambda: [eng.generate(st, sd, a.new, ()) for st, sd in zip(sts, seed)])
        toks_s = sum(len(st.ids) - a.ctx for st in sts)
        for st in sts:
            eng.truncate(st, a.ctx)
        res.update(decode_batched_tok_s=round(toks_b / tb, 1), decode_serial_tok_s=round(toks_s / ts, 1),
                   decode_speedup=round((toks_b / tb) / (toks_s / ts), 2))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
