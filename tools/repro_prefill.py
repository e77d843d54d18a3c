"""Repro: draft model, prompt -> 256-token generation -> re-prefill the
prompt + generation (suffix of 256+ tokens at start > 0)."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main() -> None:
    from paper_2504_07891_b200.backend import B200Backend
    from paper_2504_07891_b200.contract import GenerationRequest
    from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
    from paper_2504_07891_b200.shapes import get_spec
    from paper_2504_07891_b200.vocab import shared_vocab

    name = sys.argv[1] if len(sys.argv) > 1 else "r1-1.5b"
    spec = get_spec(name)
    v = shared_vocab(spec.vocab_text)
    b = B200Backend(spec, BackendRole.SMALL, max_ctx=4096 + 512)
    prompt = render_generation_prompt(v.problem(64, 0), "")
    r = b.generate_step(GenerationRequest(prompt=prompt, max_tokens=256, stop=()))
    print("gen1", r.token_count, flush=True)
    r2 = b.generate_step(GenerationRequest(prompt=prompt + r.text, max_tokens=256, stop=()))
    print("gen2", r2.token_count, flush=True)
    r3 = b.generate_step(GenerationRequest(prompt=prompt + r.text + r2.text + " ".join(v.words[100:400]) + " ",
                                           max_tokens=8, stop=()))
    print("gen3", r3.token_count, flush=True)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
