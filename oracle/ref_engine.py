"""CPU oracle engine + backend -- TEST INFRASTRUCTURE ONLY (see ref_model.py).

``RefEngine`` answers the same engine calls as the product's native engine
(``paper_2504_07891_b200/backend.py``) with the fp32 CPU decoder, and
restates the reference's judge readout literally: build the first-position
top-10 ``{token_text: logprob}`` table exactly as an OpenAI-compatible server
returns it for ``logprobs=10`` (``http.py:162-169``), take the greedy token's
text as the sampled text, and hand both to ``extract_score``
(``base.py:106-126``, mirrored in ``contract.extract_score`` and pinned
against the reference's own known answers).
"""

from __future__ import annotations

from typing import Sequence

import torch

from paper_2504_07891_b200 import contract
from paper_2504_07891_b200.domain import BackendProfile, BackendRole
from paper_2504_07891_b200.host import Readout, Stream, ModelBackend, finish_of
from paper_2504_07891_b200.shapes import ModelSpec, make_weights
from paper_2504_07891_b200.vocab import CLASS_END_THINK, CLASS_STOP, Vocab

from .ref_model import RefModel, argmax_margin, masked

TOP_LOGPROBS = 10


def top_logprobs_table(logits: torch.Tensor, vocab: Vocab, k: int = TOP_LOGPROBS) -> dict[str, float]:
    """Ordered top-k {token text: logprob}; exact ties rank the lower id first."""
    lp = torch.log_softmax(logits.to(torch.float64), dim=-1)
    # stable descending order: sort by (-logprob, id)
    order = torch.argsort(-lp, stable=True)[:k]
    return {vocab.render_one(int(i)): float(lp[i]) for i in order}


def judge_readout(logits: torch.Tensor, vocab: Vocab, threshold: int) -> Readout:
    logits = masked(logits, vocab.n_text)
    table = top_logprobs_table(logits, vocab)
    arg, margin = argmax_margin(logits)
    try:
        score = contract.extract_score(table, vocab.render_one(arg)).value
    except contract.ScoreParseFailure:
        score = -1
    return Readout(score=score, accept=score >= 0 and score >= threshold, flags=0,
                   margin=margin, argmax=arg)


class RefEngine:
    def __init__(self, spec: ModelSpec, weights: dict[str, torch.Tensor], vocab: Vocab,
                 exact_fp32: bool = False) -> None:
        self.spec = spec
        self.vocab = vocab
        self.model = RefModel(spec, weights, exact_fp32=exact_fp32)
        self.margins: list[float] = []

    def attach(self, stream: Stream) -> None:
        stream.handle = self.model.new_cache()

    def truncate(self, stream: Stream, keep: int) -> None:
        RefModel.truncate(stream.handle, keep)
        del stream.ids[keep:]

    def generate(self, stream: Stream, suffix: Sequence[int], max_new: int,
                 stop: tuple[str, ...]) -> tuple[list[int], int]:
        classes = self.vocab.token_classes(stop, self.spec.vocab_rows)
        logits = self.model.forward(stream.handle, list(suffix))
        stream.ids.extend(suffix)
        gen: list[int] = []
        while True:
            t, m = argmax_margin(masked(logits, self.vocab.n_text))
            self.margins.append(m)
            gen.append(t)
            if classes[t] in (CLASS_STOP, CLASS_END_THINK) or len(gen) >= max_new:
                break
            logits = self.model.forward(stream.handle, [t])
            stream.ids.append(t)
        return gen, finish_of(gen, classes)

    def score(self, stream: Stream, suffix: Sequence[int], threshold: int) -> Readout:
        logits = self.model.forward(stream.handle, list(suffix))
        stream.ids.extend(suffix)
        return judge_readout(logits, self.vocab, threshold)

    def prefill(self, stream: Stream, suffix: Sequence[int]) -> None:
        self.model.forward(stream.handle, list(suffix))
        stream.ids.extend(suffix)

    def verify_tokens(self, stream: Stream, suffix: Sequence[int]) -> tuple[list[int], list[float]]:
        logits = self.model.forward(stream.handle, list(suffix), last_only=False)
        stream.ids.extend(suffix)
        out = [argmax_margin(masked(row, self.vocab.n_text)) for row in logits]
        return [t for t, _ in out], [m for _, m in out]

    # multi-sequence calls: the oracle answers them one sequence at a time
    def score_batch(self, streams, suffixes, threshold: int) -> list[Readout]:
        return [self.score(s, suf, threshold) for s, suf in zip(streams, suffixes)]

    def step_batch(self, streams, feeds, room: int = 0) -> list[int]:
        out = []
        for st, f in zip(streams, feeds):
            logits = self.model.forward(st.handle, list(f))
            st.ids.extend(f)
            t, m = argmax_margin(masked(logits, self.vocab.n_text))
            self.margins.append(m)
            out.append(t)
        return out

    def generate_batch(self, streams, suffixes, max_new: int, stop: tuple[str, ...]):
        return [self.generate(s, suf, max_new, stop) for s, suf in zip(streams, suffixes)]

    def logits_teacher_forced(self, ids: Sequence[int]) -> torch.Tensor:
        """[n, V] logits of every position of ``ids`` from an empty cache."""
        cache = self.model.new_cache()
        return self.model.forward(cache, list(ids), last_only=False)


def oracle_backend(model_name: str, role: BackendRole, seed: int = 0, vocab: Vocab | None = None,
                   threshold: int = 7, types=None, record: bool = False,
                   exact_fp32: bool = False, n_streams: int = 4) -> ModelBackend:
    from paper_2504_07891_b200.shapes import get_spec
    from paper_2504_07891_b200.vocab import shared_vocab

    spec = get_spec(model_name)
    vocab = vocab or shared_vocab(spec.vocab_text)
    engine = RefEngine(spec, make_weights(spec, seed), vocab, exact_fp32=exact_fp32)
    T = types
    prof_cls = T.BackendProfile if T else BackendProfile
    role_cls = T.BackendRole if T else BackendRole
    profile = prof_cls(name=f"oracle-{model_name}", role=role_cls(role.value),
                       decode_s_per_token=1e-3, prefill_tokens_per_s=1e3)
    return ModelBackend(engine, vocab, profile, threshold=threshold, types=types,
                        record=record, n_streams=n_streams)
