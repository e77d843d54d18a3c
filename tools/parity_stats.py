"""Print GPU-vs-oracle logit error statistics next to the oracle's own
fp32-vs-fp64 noise floor (tiny models), for the current SR_* env settings."""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402


def main() -> None:
    from oracle.ref_model import RefModel
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
    from paper_2504_07891_b200.shapes import get_spec, make_weights
    from paper_2504_07891_b200.vocab import shared_vocab

    for name in sys.argv[1:] or ["tiny-draft", "tiny-base"]:
        spec = get_spec(name)
        v = shared_vocab(spec.vocab_text)
        w = make_weights(spec, 0)
        ids = v.encode(render_generation_prompt(v.problem(64, 1), "")) * 4
        a, b = RefModel(spec, w), RefModel(spec, w, dtype=torch.float64)
        la = a.forward(a.new_cache(), ids, last_only=False)[:, : v.n_text]
        lb = b.forward(b.new_cache(), ids, last_only=False)[:, : v.n_text].float()
        gpu = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=2048)
        s = gpu.pool.streams[0]
        got = gpu.engine.forward_logits(s, ids).cpu()[:, : v.n_text]
        e, f = (got - la).abs(), (la - lb).abs()
        pe, pf = e.max(-1).values, f.max(-1).values
        worst = torch.topk(pe, 8).indices.tolist()
        print(json.dumps({"model": name, "worst_positions": worst,
                          "their_err": [round(float(pe[i]), 4) for i in worst],
                          "floor_there": [round(float(pf[i]), 4) for i in worst],
                          "err_by_64": [round(float(pe[i:i + 64].mean()), 5) for i in range(0, len(ids), 64)],
                          "floor_by_64": [round(float(pf[i:i + 64].mean()), 5) for i in range(0, len(ids), 64)]}))
        print(json.dumps({"model": name, "gpu_vs_oracle": {"max": e.max().item(), "mean": e.mean().item()},
                          "oracle32_vs_64": {"max": f.max().item(), "mean": f.mean().item()},
                          "gpu_vs_oracle64": {"max": (got - lb).abs().max().item(),
                                              "mean": (got - lb).abs().mean().item()}}), flush=True)


if __name__ == "__main__":
    main()
