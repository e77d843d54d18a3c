"""Fine-grained bring-up probe: every native call is followed by a
synchronize and a flushed print, and faulthandler dumps the Python stack if
anything stalls, so a hang is located to one call."""

from __future__ import annotations

import faulthandler
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
faulthandler.dump_traceback_later(int(os.environ.get("PROBE_DUMP_S", "60")), repeat=True)

import torch  # noqa: E402

T0 = time.time()


def say(*a):
    print(f"[{time.time() - T0:7.2f}s]", *a, flush=True)


def main(which: str) -> None:
    from oracle.ref_engine import RefEngine
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.contract import GenerationRequest, VerificationRequest
    from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
    from paper_2504_07891_b200.shapes import get_spec, make_weights
    from paper_2504_07891_b200.vocab import shared_vocab

    spec = get_spec(which)
    v = shared_vocab(spec.vocab_text)
    w = make_weights(spec, 0)
    say("weights ready")
    gpu = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024)
    torch.cuda.synchronize()
    say("model created")
    ref = RefEngine(spec, w, v)
    ids = v.encode(render_generation_prompt(v.problem(64, 1), ""))
    s = gpu.pool.streams[0]
    out = gpu.engine.forward_logits(s, ids[:8], all_rows=False)
    torch.cuda.synchronize()
    say("forward_logits(8, last) ok", float(out.abs().max()))
    gpu.engine.truncate(s, 0)
    out = gpu.engine.forward_logits(s, ids).cpu()
    want = ref.logits_teacher_forced(ids)
    say("forward_logits(all) maxabs", float((out[:, :v.n_text] - want[:, :v.n_text]).abs().max()),
        "argmax agree", float((out[:, :v.n_text].argmax(-1) == want[:, :v.n_text].argmax(-1)).float().mean()))
    r = gpu.generate_step(GenerationRequest(prompt=render_generation_prompt(v.problem(64, 2), ""),
                                            max_tokens=1, stop=()))
    say("generate max_tokens=1 ok", repr(r.text), r.finish_reason)
    r = gpu.generate_step(GenerationRequest(prompt=render_generation_prompt(v.problem(64, 2), ""),
                                            max_tokens=8, stop=()))
    say("generate max_tokens=8 ok", repr(r.text), r.finish_reason, gpu.engine.last_margins)
    sc = gpu.score_step(VerificationRequest("a b c", "d e f ", "g h "))
    say("score ok", sc)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["tiny-base"]:
        say("==", name)
        main(name)
    say("done")
