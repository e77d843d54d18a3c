"""Token-level speculation on the device (``sr_verify_tokens``): the base
model's steps generated with a draft proposing tokens equal plain greedy
device decoding, up to flagged near-ties (the verify pass uses the tensor-core
prefill path, plain decode the persistent GEMV kernel; tolerance: tests/tolerance.py)."""

import pytest

from oracle.ref_engine import RefEngine
from paper_2504_07891_b200.contract import GenerationRequest
from paper_2504_07891_b200.domain import DEFAULT_STEP_STOP_MARKERS, BackendRole, render_generation_prompt
from paper_2504_07891_b200.shapes import get_spec, make_weights
from paper_2504_07891_b200.vocab import shared_vocab

from tolerance import floor_tol

pytestmark = pytest.mark.gpu
TOL = floor_tol("tiny-base")  # tests/tolerance.py


@pytest.mark.parametrize("draft_name", ["tiny-draft", "tiny-base"])
def test_device_speculation_matches_plain_decode(cuda, draft_name):
    from paper_2504_07891_b200.backend import B200Backend

    spec = get_spec("tiny-base")
    w = make_weights(spec, 0)
    v = shared_vocab(spec.vocab_text)
    plain = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024)
    fast = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024)
    dspec = get_spec(draft_name)
    draft = B200Backend(dspec, BackendRole.SMALL, weights=w if draft_name == "tiny-base" else None,
                        max_ctx=1024)
    fast.attach_speculator(draft, gamma=5)
    ref = RefEngine(spec, w, v)
    identical = 0
    for p in range(4):
        prompt = render_generation_prompt(v.problem(64, 50 + p), "")
        req = GenerationRequest(prompt=prompt, max_tokens=40, stop=DEFAULT_STEP_STOP_MARKERS)
        a, b = plain.generate_step(req), fast.generate_step(req)
        if a.text == b.text:
            assert a.finish_reason == b.finish_reason
            identical += 1
            continue
        ia, ib = v.encode(a.text), v.encode(b.text)
        k = next(i for i, (x, y) in enumerate(zip(ia, ib)) if x != y)
        lg = ref.logits_teacher_forced(v.encode(prompt) + ia[:k])[-1][: v.n_text]
        assert abs(float(lg[ia[k]] - lg[ib[k]])) < TOL, (p, k)
    assert identical >= 3
    st = fast.spec_stats
    rate = st["accepted"] / max(1, st["proposed"])
    print(f"speculation with {draft_name}: {st}, acceptance {rate:.2f}")
    assert (rate > 0.8) if draft_name == "tiny-base" else True
