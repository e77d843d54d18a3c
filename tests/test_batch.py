"""Several independent requests per device pass: the batched
``score_steps`` / ``generate_steps`` of ``ModelBackend`` return what the
per-request calls return.  CPU: oracle engine (host logic: distinct streams,
prefix reuse, result mapping)."""

import numpy as np
import pytest

from oracle.ref_engine import oracle_backend
from paper_2504_07891_b200.contract import GenerationRequest, VerificationRequest
from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
from paper_2504_07891_b200.vocab import shared_vocab


def _requests(v, n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        w = [v.words[int(x)] for x in rng.integers(16, v.n_text, size=90)]
        out.append(VerificationRequest(" ".join(w[:40]), " ".join(w[40:80]) + " ", " ".join(w[80:]) + " "))
    return out


def test_score_steps_match_score_step():
    base = oracle_backend("tiny-base", BackendRole.BASE, n_streams=4)
    ref = oracle_backend("tiny-base", BackendRole.BASE, n_streams=4)
    reqs = _requests(shared_vocab(base.engine.spec.vocab_text), 3, 1)
    got = base.score_steps(reqs)
    for r, g in zip(reqs, got):
        try:
            want = ref.score_step(r).value
        except Exception as exc:
            assert type(exc).__name__ == type(g).__name__ == "ScoreParseFailure"
            continue
        assert g.value == want
    # a second batch sharing the prefixes reuses the streams (fresh rows only)
    got2 = base.score_steps(reqs)
    assert [getattr(x, "value", None) for x in got2] == [getattr(x, "value", None) for x in got]


def test_generate_steps_match_generate_step():
    small = oracle_backend("tiny-draft", BackendRole.SMALL, n_streams=4)
    ref = oracle_backend("tiny-draft", BackendRole.SMALL, n_streams=4)
    v = shared_vocab(small.engine.spec.vocab_text)
    reqs = [GenerationRequest(prompt=render_generation_prompt(v.problem(32, k), ""), max_tokens=12,
                              stop=("\n\n",)) for k in range(3)]
    got = small.generate_steps(reqs)
    for r, g in zip(reqs, got):
        w = ref.generate_step(r)
        assert (g.text, g.token_count, g.finish_reason) == (w.text, w.token_count, w.finish_reason)


def test_batch_needs_distinct_streams():
    base = oracle_backend("tiny-base", BackendRole.BASE, n_streams=2)
    reqs = _requests(shared_vocab(base.engine.spec.vocab_text), 3, 2)
    with pytest.raises(ValueError, match="KV streams"):
        base.score_steps(reqs)
