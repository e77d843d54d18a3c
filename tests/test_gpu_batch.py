"""Multi-sequence passes on the B200: ``sr_score_batch`` and
``sr_step_batch`` against the per-sequence device calls and the CPU oracle.

Batching changes only the row count of the GEMMs (tiling and split-K order),
so results must agree except where the top-2 margin is below the parity
tolerance (flagged near-ties)."""

import dataclasses

import numpy as np
import pytest
import torch

from oracle.ref_engine import RefEngine, judge_readout
from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt
from paper_2504_07891_b200.shapes import get_spec, make_weights
from paper_2504_07891_b200.vocab import shared_vocab

from tolerance import floor_tol

pytestmark = pytest.mark.gpu
TOL = floor_tol("tiny-base")  # tests/tolerance.py


def _suffixes(v, n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    return [[int(x) for x in rng.integers(16, v.n_text, size=int(rng.integers(lo, hi)))]
            for _ in range(n)]


@pytest.fixture(scope="module")
def tiny(cuda):
    from paper_2504_07891_b200.backend import B200Backend

    a = B200Backend("tiny-base", BackendRole.BASE, max_ctx=1024, n_streams=8)
    b = B200Backend("tiny-base", BackendRole.BASE, max_ctx=1024, n_streams=8)
    return a, b, shared_vocab(a.engine.spec.vocab_text)


def test_score_batch_matches_single(tiny):
    a, b, v = tiny
    # two rounds: fresh streams, then appended suffixes on the cached contexts
    for rnd, (lo, hi) in enumerate([(60, 200), (5, 40)]):
        sufs = _suffixes(v, 6, lo, hi, 10 + rnd)
        got = a.engine.score_batch(a.pool.streams[:6], sufs, 7)
        for k, suf in enumerate(sufs):
            want = b.engine.score(b.pool.streams[k], suf, 7)
            if (got[k].score, got[k].accept) != (want.score, want.accept):
                assert want.margin < TOL, (rnd, k, got[k], want)
        assert [len(s.ids) for s in a.pool.streams[:6]] == [len(s.ids) for s in b.pool.streams[:6]]


def test_generate_batch_matches_single(tiny):
    from paper_2504_07891_b200.backend import B200Backend

    s = B200Backend("tiny-draft", BackendRole.SMALL, max_ctx=1024, n_streams=8)
    v = shared_vocab(s.engine.spec.vocab_text)
    prompts = [v.encode(render_generation_prompt(v.problem(48, 30 + k), "")) for k in range(5)]
    outs = s.engine.generate_batch(s.pool.streams[:5], prompts, 40, ())
    for k, p in enumerate(prompts):
        st = s.pool.streams[5 + (k % 3)]
        s.engine.truncate(st, 0)
        gen, fin = s.engine.generate(st, p, 40, ())
        margins = s.engine.last_margins
        got = outs[k][0]
        n = min(len(gen), len(got))
        first = next((i for i in range(n) if gen[i] != got[i]), None)
        if first is None:
            assert len(gen) == len(got) and outs[k][1] == fin
        else:
            assert margins[first] < TOL, (k, first, margins[first])


@pytest.mark.parametrize("model", ["qwen2.5-7b", "qwq-32b"])
def test_score_batch_fullwidth_vs_oracle(cuda, model):
    """Real 7B / 32B widths (2 layers): 8 verify-sized sequences in one pass,
    each readout against the fp32 oracle."""
    from paper_2504_07891_b200.backend import B200Backend

    full = get_spec(model)
    spec = dataclasses.replace(full, n_layers=2)
    w = make_weights(full, 0, layers=[0, 1])
    v = shared_vocab(spec.vocab_text)
    gpu = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=512, n_streams=8)
    ref = RefEngine(spec, w, v)
    sufs = _suffixes(v, 8, 60, 100, 44)
    got = gpu.engine.score_batch(gpu.pool.streams, sufs, 7)
    agree = 0
    for k, suf in enumerate(sufs):
        want = judge_readout(ref.model.forward(ref.model.new_cache(), suf), v, 7)
        if got[k].score == want.score:
            agree += 1
        else:
            assert want.margin < TOL, (k, got[k], want)
    assert agree >= 6


def test_batch_passes_beyond_max_tokens(cuda):
    """Sequences longer than one pass and batches whose rows exceed max_tokens:
    split into passes / the chunked single-sequence path, same results."""
    from paper_2504_07891_b200.backend import B200Backend

    a = B200Backend("tiny-base", BackendRole.BASE, max_ctx=2048, n_streams=6, max_tokens=128)
    b = B200Backend("tiny-base", BackendRole.BASE, max_ctx=2048, n_streams=6, max_tokens=128)
    v = shared_vocab(a.engine.spec.vocab_text)
    sufs = _suffixes(v, 5, 40, 300, 77)  # some longer than a 128-row pass
    got = a.engine.score_batch(a.pool.streams[:5], sufs, 7)
    for k, suf in enumerate(sufs):
        want = b.engine.score(b.pool.streams[k], suf, 7)
        if (got[k].score, got[k].accept) != (want.score, want.accept):
            assert want.margin < TOL, (k, got[k], want)
    # generation from long prompts: the prompt goes through the chunked path first
    s = B200Backend("tiny-draft", BackendRole.SMALL, max_ctx=2048, n_streams=6, max_tokens=128)
    prompts = _suffixes(v, 3, 150, 400, 78)
    outs = s.engine.generate_batch(s.pool.streams[:3], prompts, 12, ())
    for k, p in enumerate(prompts):
        st = s.pool.streams[3 + k]
        gen, _ = s.engine.generate(st, p, 12, ())
        first = next((i for i in range(min(len(gen), len(outs[k][0]))) if gen[i] != outs[k][0][i]), None)
        if first is not None:
            assert s.engine.last_margins[first] < TOL, (k, first)
