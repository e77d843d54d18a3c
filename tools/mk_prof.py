"""Phase timeline of the persistent decode kernel (SR_MK_PROF=1).

    python tools/mk_prof.py r1-1.5b --ctx 2048

Prints, for the first decoded token, the mean duration of each phase step
over the layers (CTA 0's view, globaltimer ns) and the LM-head tail."""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SR_MK_PROF"] = "1"

import torch  # noqa: E402

NAMES = ["qkv_prologue", "qkv_gemv", "sync_qkv", "attention", "sync_attn", "combine", "sync_comb",
         "o_stage",
         "o_gemv", "sync_o", "gu_prologue", "gu_gemv", "sync_gu", "d_stage", "d_gemv", "sync_d"]
E = len(NAMES)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--ctx", type=int, default=2048)
    a = ap.parse_args()
    from paper_2504_07891_b200 import native
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.shapes import get_spec

    spec = get_spec(a.model)
    b = B200Backend(spec, BackendRole.BASE, max_ctx=a.ctx + 128)
    g = torch.Generator().manual_seed(0)
    ctx = torch.randint(16, spec.vocab_text, (a.ctx,), generator=g).tolist()
    s = b.pool.streams[0]
    out = {}
    for rep in range(2):
        b.engine.truncate(s, 0)
        b.engine.generate(s, ctx, 4, ())
    buf = (C.c_uint64 * 2048)()
    native.check("sr_debug_profile", native.load().sr_debug_profile(b.device_model.handle, buf, 2048))
    ev = list(buf)
    L = spec.n_layers
    n = 1 + E * L + 4
    t = ev[:n]
    per = {k: 0.0 for k in NAMES}
    for l in range(L):
        base = 1 + E * l
        for i, name in enumerate(NAMES):
            prev = t[base + i - 1]
            per[name] += (t[base + i] - prev) / 1e3
    out["per_layer_us"] = {k: round(v / L, 3) for k, v in per.items()}
    tail = t[1 + E * L:]
    last = t[E * L]
    out["lm_us"] = {"prologue": round((tail[0] - last) / 1e3, 2),
                    "gemv": round((tail[1] - tail[0]) / 1e3, 2),
                    "sync": round((tail[2] - tail[1]) / 1e3, 2),
                    "select": round((tail[3] - tail[2]) / 1e3, 2)}
    out["token_us"] = round((t[n - 1] - t[0]) / 1e3, 1)
    import statistics
    att = ev[1280:1280 + 148]
    last = ev[1440:1440 + 148]
    busy = [x / 1e3 for x in att if x > 0]
    if busy:
        out["attn_cta_us"] = {"n": len(busy), "min": round(min(busy), 2),
                              "median": round(statistics.median(busy), 2),
                              "max": round(max(busy), 2),
                              "last_split_max": round(max([x / 1e3 for x, f in zip(att, last) if f] or [0]), 2)}
    sub = [x for x in ev[1600:1632] if x > 0]
    out["attn_cta0_steps_us"] = [round((b - a) / 1e3, 2) for a, b in zip(sub, sub[1:])]
    for name, base in (("qkv_prologue_steps_us", 1640), ("gu_prologue_steps_us", 1650)):
        st = ev[base:base + 4]
        if all(x > 0 for x in st):  # loads | block sum | normalise + store
            out[name] = [round((b - a) / 1e3, 2) for a, b in zip(st, st[1:])]
    out["model"] = a.model
    out["ctx"] = a.ctx
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
