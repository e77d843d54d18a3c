"""Verify-pass timing (K6 + K7 + K8): prefill a context, then score `--m`-token
suffixes on top of it (rolled back after each call, as the base-verify stream
does).  Prints CUDA-event ms per call and the HBM / tensor rooflines (SURVEY
§8d).  Under ncu, the last call's kernels are the tail of the launch list.

    python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 --reps 5
"""

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
    ap.add_argument("--m", type=int, default=80)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--max-tokens", type=int, default=256, help="largest prefill chunk")
    a = ap.parse_args()
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.shapes import get_spec

    spec = get_spec(a.model)
    b = B200Backend(spec, BackendRole.BASE, max_ctx=a.ctx + a.m + 64, max_tokens=a.max_tokens)
    eng = b.engine
    g = torch.Generator().manual_seed(0)
    ctx = torch.randint(16, spec.vocab_text, (a.ctx,), generator=g).tolist()
    s = b.pool.streams[0]
    eng.forward_logits(s, ctx, all_rows=False)
    times = []
    from bench import ClockSampler  # nvidia-smi clocks / throttle reasons during the timed calls

    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(a.reps):
            ids = torch.randint(16, spec.vocab_text, (a.m,), generator=g).tolist()
            eng.score(s, ids, 7)
            t = eng.model.timing()
            times.append(t.prefill_ms)
            eng.truncate(s, a.ctx)
    ms = min(times)
    P = spec.body_params() + spec.head_params()
    C, M = a.ctx, a.m
    byts = 2 * P + (C + M) * spec.kv_bytes_per_token()
    flops = 2 * M * spec.body_params() + 4 * spec.n_layers * spec.n_heads * 128 * M * (C + M / 2) \
        + 2 * spec.vocab_rows * spec.d_model
    print(json.dumps({"model": a.model, "ctx": C, "m": M, "ms": round(ms, 3), "all_ms": [round(x, 3) for x in times],
                      "GBps": round(byts / (ms * 1e-3) / 1e9, 1), "TFLOPs": round(flops / (ms * 1e-3) / 1e12, 1),
                      "hbm_floor_ms": round(byts / 6552e9 * 1e3, 3),
                      "tensor_floor_ms": round(flops / 1.374e15 * 1e3, 3),
                      "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
