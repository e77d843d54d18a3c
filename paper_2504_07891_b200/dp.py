"""Request-level data parallelism over independent problems (config C5).

The reference's only parallelism is ``run_sweep`` (``bench.py:221-300``):
every (knob value x scheme x problem x repeat) trajectory is an independent
job, seeded by ``trajectory_seed(base_seed, problem_id, repeat)``
(``bench.py:216-218``) so a cell's result never depends on the knob value or
on which worker ran it.  Here the workers are GPUs (one process per GPU,
``torch.distributed``): the fixed problem set is split into contiguous
``problem_id`` blocks, each rank runs its block through its own backends
(no collective on the data path), and the per-problem records are gathered
on rank 0 at the end -- the same host-side gather as the reference's
``records`` list.  Because every trajectory depends only on its problem id,
the gathered records are identical for any world size
(``tests/test_dp.py`` runs world 1 and world 2 on CPU oracle backends).

Acceptance criterion of the sweep (``test_acceptance.py:104-113``): at
threshold 10 SpecReason rejects every draft step, so its CoT and answer must
equal the BaseOnly run (``run_vanilla`` of the base) of the same problem;
``check_forced_reject`` asserts it per problem.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, replace
from typing import Any, Sequence

from .domain import AcceptanceThreshold, EngineConfig, Scheme
from .driver import run_trajectory, run_vanilla
from .pricing import derive_seed, trajectory_seed


def problem_ids(n: int) -> list[str]:
    """The reference's problem naming (``bench.py:238``)."""
    return [f"task{i:04d}" for i in range(n)]


def partition(ids: Sequence[str], rank: int, world: int) -> list[str]:
    """Contiguous block of ``ids`` owned by ``rank`` (sizes differ by <= 1)."""
    n = len(ids)
    lo = rank * n // world
    hi = (rank + 1) * n // world
    return list(ids[lo:hi])


def problem_text(vocab: Any, problem_id: str, n_words: int = 64, base_seed: int = 0) -> str:
    """Synthetic problem statement of ``problem_id``: a function of the id
    only, never of the rank that runs it."""
    return vocab.problem(n_words, derive_seed("problem", base_seed, problem_id) & ((1 << 32) - 1))


@dataclass(frozen=True)
class Record:
    problem_id: str
    repeat: int
    scheme: str
    knob_value: int
    thinking_tokens: int
    accepted_fraction: float | None
    rejected_count: int
    cot_digest: str
    answer_digest: str
    latency_s: float

    def key(self) -> tuple:
        return (self.scheme, self.knob_value, self.problem_id, self.repeat)

    def outcome(self) -> tuple:
        """Everything but the measured latency (which is wall clock)."""
        return (self.thinking_tokens, self.accepted_fraction, self.rejected_count,
                self.cot_digest, self.answer_digest)


def _digest(text: str) -> str:
    return hashlib.sha1(text.encode("utf-8")).hexdigest()[:16]


def run_scheme(scheme: Scheme, config: EngineConfig, problem: str, small: Any, base: Any):
    """``run_scheme`` (``bench.py:196-213``) for the two schemes of the sweep."""
    if scheme == Scheme.BASE_ONLY:
        return run_vanilla(config, problem, base)
    if scheme == Scheme.SPEC_REASON:
        return run_trajectory(replace(config, hierarchical=False), problem, small, base)
    raise ValueError(f"unsupported scheme {scheme}")


def cold_start(*backends: Any) -> None:
    """Drop every cached K/V stream so a trajectory's arithmetic depends on
    its problem only: otherwise a later problem would reuse K/V an earlier
    one left (the verification template's shared head), computed in other
    prefill chunks, and results would depend on which problems a rank ran
    before (the partition)."""
    for b in backends:
        pool = getattr(b, "pool", None)
        if pool is not None:
            for s in pool.streams:
                b.engine.truncate(s, 0)


def run_partition(ids: Sequence[str], small: Any, base: Any, base_config: EngineConfig,
                  thresholds: Sequence[int], *, repeats: int = 1,
                  schemes: Sequence[Scheme] = (Scheme.SPEC_REASON,),
                  problem_words: int = 64) -> list[Record]:
    """Every (threshold x scheme x problem x repeat) trajectory of this rank's
    problems.  BaseOnly does not depend on the threshold: it runs once per
    problem, recorded with knob value -1."""
    out: list[Record] = []
    jobs = []
    for scheme in schemes:
        values = [-1] if scheme == Scheme.BASE_ONLY else list(thresholds)
        jobs += [(v, scheme, pid, r) for v in values for pid in ids for r in range(repeats)]
    for value, scheme, pid, rep in jobs:
        cold_start(small, base)
        cfg = base_config
        if value >= 0:
            cfg = replace(cfg, threshold=AcceptanceThreshold(value))
            if hasattr(base, "threshold"):
                base.threshold = value
        cfg = replace(cfg, seed=trajectory_seed(base_config.seed, pid, rep))
        res = run_scheme(scheme, cfg, problem_text(small.vocab, pid, problem_words), small, base)
        m = res.metrics
        out.append(Record(pid, rep, scheme.value, value, m.thinking_tokens, m.accepted_fraction,
                          m.rejected_count, _digest(res.state.cot_text()),
                          _digest(res.state.final_answer or ""), m.latency_s))
    return out


def gather(records: list[Record], dist: Any = None) -> list[Record]:
    """All ranks' records on every rank (gloo/nccl object all-gather), sorted
    like the reference's ``records.sort`` (``bench.py:289``)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        box: list = [None] * dist.get_world_size()
        dist.all_gather_object(box, records)
        records = [r for part in box for r in part]
    return sorted(records, key=lambda r: (r.scheme, str(r.knob_value), r.problem_id, r.repeat))


def check_forced_reject(records: Sequence[Record]) -> int:
    """Threshold 10 SpecReason == BaseOnly, per problem (CoT and answer);
    returns the number of problems checked."""
    base = {(r.problem_id, r.repeat): r for r in records if r.scheme == Scheme.BASE_ONLY.value}
    n = 0
    for r in records:
        if r.scheme == Scheme.SPEC_REASON.value and r.knob_value == 10:
            b = base.get((r.problem_id, r.repeat))
            if b is None:
                continue
            if (r.cot_digest, r.answer_digest, r.thinking_tokens) != (
                    b.cot_digest, b.answer_digest, b.thinking_tokens):
                raise AssertionError(f"{r.problem_id}: threshold 10 differs from BaseOnly")
            if r.accepted_fraction not in (0.0, None):
                raise AssertionError(f"{r.problem_id}: threshold 10 accepted a draft step")
            n += 1
    return n


def cells(records: Sequence[Record]) -> dict:
    """Per (scheme, knob value): mean accepted fraction, CoT tokens and the
    CoT tokens/s of the cell (thinking tokens / latency summed)."""
    out: dict = {}
    for r in records:
        c = out.setdefault(f"{r.scheme}@{r.knob_value}", {"n": 0, "tokens": 0, "latency_s": 0.0,
                                                          "accepted": []})
        c["n"] += 1
        c["tokens"] += r.thinking_tokens
        c["latency_s"] += r.latency_s
        if r.accepted_fraction is not None:
            c["accepted"].append(r.accepted_fraction)
    for c in out.values():
        acc = c.pop("accepted")
        c["accepted_fraction"] = round(sum(acc) / len(acc), 4) if acc else None
        c["cot_tok_s"] = round(c["tokens"] / c["latency_s"], 2) if c["latency_s"] > 0 else None
    return out
