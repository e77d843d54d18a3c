"""Tensor-parallel device paths on one GPU.

World size 2 over NVLink peer memory (``PeerTransport``): two ranks of one
process share the GPU (72 persistent-decode CTAs each, so both kernels are
co-resident) and drive the same calls from two threads on two streams.  The
fused tensor-parallel decode kernel (in-kernel exchange of the row-parallel
deltas and the vocab-parallel greedy merge) and the one-shot peer collectives
of prefill and the judge readout must give both ranks identical results,
equal to the unsharded oracle's up to flagged near-ties.

World size 1 over NCCL:

With a communicator attached the runtime takes every TP code path: split
partials all-reduced into a delta before the residual add (prefill), the
host-driven decode loop with an all-reduce after O and down and a
vocab-parallel greedy merge, and the judge readout from all-reduced digit
rank counts.  At world size 1 these must reproduce the single-GPU path
(greedy tokens equal except at flagged near-ties, identical scores and
accept bits).  The world > 1 decomposition itself is checked on CPU ranks
(tests/test_tp.py).
"""

import numpy as np
import pytest
import torch

from oracle.ref_engine import RefEngine
from paper_2504_07891_b200.contract import VerificationRequest
from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
from paper_2504_07891_b200.shapes import get_spec, make_weights
from paper_2504_07891_b200.vocab import shared_vocab

from tolerance import floor_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair(cuda):
    from paper_2504_07891_b200.backend import B200Backend, TensorParallel

    spec = get_spec("tiny-base")
    w = make_weights(spec, 0)
    tp = TensorParallel.single()
    a = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024)
    b = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024, tp=tp)
    return spec, w, a, b


def test_tp1_prefill_logits_match(pair):
    spec, w, a, b = pair
    v = shared_vocab(spec.vocab_text)
    ids = v.encode(render_generation_prompt(v.problem(64, 9), ""))
    la = a.engine.forward_logits(a.pool.streams[0], ids).cpu()
    lb = b.engine.forward_logits(b.pool.streams[0], ids).cpu()
    assert (la - lb).abs().max().item() < 2e-2


def test_tp1_decode_matches_or_flags(pair):
    spec, w, a, b = pair
    v = shared_vocab(spec.vocab_text)
    ref = RefEngine(spec, w, v)
    for p in range(3):
        ids = v.encode(render_generation_prompt(v.problem(64, 20 + p), ""))
        ga, _ = a.engine.generate(a.pool.streams[1], ids, 32, ())
        gb, _ = b.engine.generate(b.pool.streams[1], ids, 32, ())
        a.engine.truncate(a.pool.streams[1], 0)
        b.engine.truncate(b.pool.streams[1], 0)
        assert len(gb) == 32
        lg = ref.logits_teacher_forced(ids + gb[:-1])[len(ids) - 1:, : v.n_text]
        for k, t in enumerate(gb):
            top = int(lg[k].argmax())
            assert t == top or float(lg[k][top] - lg[k][t]) < floor_tol("tiny-base"), (p, k)


def test_tp1_judge_readout_matches(pair):
    spec, w, a, b = pair
    v = shared_vocab(spec.vocab_text)
    rng = np.random.default_rng(1)
    same = 0
    for i in range(12):
        words = [v.words[int(x)] for x in rng.integers(16, v.n_text, size=160)]
        req = VerificationRequest(" ".join(words[:64]), " ".join(words[64:136]) + " ",
                                  " ".join(words[136:]) + " ")
        out = []
        for be in (a, b):
            try:
                out.append(be.score_step(req).value)
            except Exception as exc:
                assert type(exc).__name__ == "ScoreParseFailure"
                out.append(-1)
        same += out[0] == out[1]
    assert same >= 11


def _on_ranks(backends, fn):
    """Run fn(rank_backend) on every rank concurrently (own thread + stream)."""
    import threading

    out, err = [None] * len(backends), []

    def work(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(backends[r])
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001
            err.append(exc)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(len(backends))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "a tensor-parallel rank hung"
    if err:
        raise err[0]
    return out


@pytest.fixture(scope="module")
def tp2(cuda):
    import os

    from paper_2504_07891_b200.backend import B200Backend, TensorParallel

    spec = get_spec("tiny-base")
    w = make_weights(spec, 0)
    old = os.environ.get("SR_MK_CTAS")
    os.environ["SR_MK_CTAS"] = "72"
    try:
        tps = TensorParallel.local_group(2)
        ranks = [B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024, tp=tps[r],
                             record=True) for r in range(2)]
    finally:
        if old is None:
            os.environ.pop("SR_MK_CTAS", None)
        else:
            os.environ["SR_MK_CTAS"] = old
    return spec, w, ranks


def test_tp2_peer_decode_matches_oracle(tp2):
    from paper_2504_07891_b200.contract import GenerationRequest

    spec, w, ranks = tp2
    v = shared_vocab(spec.vocab_text)
    ref = RefEngine(spec, w, v)
    tol = floor_tol("tiny-base")
    for p in range(3):
        prompt = render_generation_prompt(v.problem(64, 30 + p), "")
        req = GenerationRequest(prompt=prompt, max_tokens=40, stop=())
        a, b = _on_ranks(ranks, lambda be: be.generate_step(req))
        assert a.text == b.text and a.token_count == 40
        ids = v.encode(prompt)
        gen = v.encode(a.text)
        lg = ref.logits_teacher_forced(ids + gen[:-1])[len(ids) - 1:, : v.n_text]
        for k, t in enumerate(gen):
            top = int(lg[k].argmax())
            assert t == top or float(lg[k][top] - lg[k][t]) < tol, (p, k, t, top)


def test_tp2_peer_readout(tp2):
    from oracle.ref_engine import judge_readout
    from oracle.tree_oracle import readout_ambiguity

    spec, w, ranks = tp2
    v = shared_vocab(spec.vocab_text)
    ref = RefEngine(spec, w, v)
    rng = np.random.default_rng(7)
    for i in range(6):
        words = [v.words[int(x)] for x in rng.integers(16, v.n_text, size=160)]
        req = VerificationRequest(" ".join(words[:64]), " ".join(words[64:136]) + " ",
                                  " ".join(words[136:]) + " ")

        def score(be):
            try:
                return be.score_step(req).value
            except Exception as exc:  # noqa: BLE001
                assert type(exc).__name__ == "ScoreParseFailure"
                return -1

        a, b = _on_ranks(ranks, score)
        assert a == b
        ids = ranks[0].calls[-1]["prompt_ids"]
        lg = ref.model.forward(ref.model.new_cache(), ids)
        want = judge_readout(lg, v, 7)
        assert a == want.score or readout_ambiguity(lg, v.n_text) < floor_tol("tiny-base")
