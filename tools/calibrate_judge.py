"""Measure the judge-circuit offsets of a base model (see shapes.py).

    python tools/calibrate_judge.py tiny-base            # CPU oracle (tiny shapes)
    python tools/calibrate_judge.py qwen2.5-7b --gpu      # on the B200 (full shapes)

Prints the offsets to paste into shapes.MODELS and the score histogram over
the calibration prompts before/after."""

from __future__ import annotations

import collections
import dataclasses
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_07891_b200.shapes import (get_spec, judge_calibration_prompts,  # noqa: E402
                                          judge_offsets_update, make_weights)


class GpuJudge:
    """Base model on the B200; only the LM head depends on the offsets, so it
    is regenerated in place between iterations (the 32B fits once, not twice)."""

    def __init__(self, spec):
        from paper_2504_07891_b200.backend import B200Backend
        from paper_2504_07891_b200.domain import BackendRole

        self.b = B200Backend(spec, BackendRole.BASE, weights=make_weights(spec, 0, device="cuda"),
                             max_ctx=8192, n_streams=1)
        self.s = self.b.pool.streams[0]

    def set_spec(self, spec):
        from paper_2504_07891_b200.shapes import make_tensor

        self.b.device_model.weights["lm_head"].copy_(make_tensor(spec, 0, "lm_head", "cuda"))

    def __call__(self, ids):
        self.b.engine.truncate(self.s, 0)
        return self.b.engine.forward_logits(self.s, ids, all_rows=False)[0].cpu()


def logits_fn_for(spec, gpu: bool):
    w = make_weights(spec, 0, device="cpu")
    from oracle.ref_model import RefModel

    m = RefModel(spec, w)
    return lambda ids: m.forward(m.new_cache(), ids)


def main() -> None:
    name = sys.argv[1]
    gpu = "--gpu" in sys.argv
    over = {}
    for flag, key in (("--digit-noise", "digit_noise"), ("--digit-gain", "digit_gain"),
                      ("--probe-gain", "probe_gain"), ("--probe-scale", "probe_scale")):
        if flag in sys.argv:
            over[key] = float(sys.argv[sys.argv.index(flag) + 1])
    spec = get_spec(name, **over)
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 24
    step = int(sys.argv[sys.argv.index("--cot-step") + 1]) if "--cot-step" in sys.argv else 25
    prompts = judge_calibration_prompts(spec, n, step, chain=spec.succ_gain > 0)
    judge = GpuJudge(spec) if gpu else None
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 4
    for it in range(iters):
        if gpu:
            judge.set_spec(spec)
            fn = judge
        else:
            fn = logits_fn_for(spec, gpu)
        rows = [fn(p) for p in prompts]
        hist = collections.Counter(int(r[:10].argmax()) for r in rows)
        import torch

        L = torch.stack([r.float() for r in rows])
        tenth = torch.topk(L[:, : spec.vocab_text], 10, dim=1).values[:, -1]
        member = (L[:, :10] >= tenth[:, None]).float().mean().item()
        dev = L[:, :10] - L[:, :10].mean(1, keepdim=True)
        print(f"  probe {L[:, spec.vocab_text].mean():.3f} digit-member frac {member:.3f} "
              f"context spread (std over prompts of centred digit logits) "
              f"{(dev - dev.mean(0)).std().item():.3f}", flush=True)
        print(f"iter {it}: offsets {spec.judge_offsets} -> argmax-digit histogram {sorted(hist.items())}",
              flush=True)
        spec = dataclasses.replace(spec, judge_offsets=judge_offsets_update(spec, rows))
    print("judge_offsets =", spec.judge_offsets)
    # one trajectory: consecutive steps share the context and differ in the
    # candidate; a judge that reads the candidate changes score step to step
    traj = judge_calibration_prompts(spec, 40, 24, chain=spec.succ_gain > 0, one_chain=True)
    if gpu:
        judge.set_spec(spec)
        fn = judge
    else:
        fn = logits_fn_for(spec, gpu)
    sc = [int(fn(p)[:10].argmax()) for p in traj]
    same = sum(a == b for a, b in zip(sc, sc[1:])) / (len(sc) - 1)
    print(f"trajectory scores {sc}  consecutive-equal {same:.2f} (independent ~0.1) "
          f"accept@7 {sum(x >= 7 for x in sc) / len(sc):.2f}", flush=True)
    print("OVERRIDE " + "".join(f"{k}={v}," for k, v in over.items())
          + "judge_offsets=" + ":".join(str(x) for x in spec.judge_offsets))


if __name__ == "__main__":
    main()
