"""SpecReason driver: draft a step, score it, accept or fall back.

Host-side mirror of the reference engine (``pkg/src/stepspec/engine.py``)
with identical observable behaviour -- same retained steps, audit copies,
trace records and latency arithmetic -- so any ``Backend`` (the B200 one, the
CPU oracle, or the reference's own simulated/HTTP backends) can be driven by
either implementation and produce the same trajectory.

Reference anchors:
  run_trajectory        engine.py:297-354
  thinking loop         engine.py:357-521
  segment_step          engine.py:114-136
  prefix ledger         engine.py:161-186 (KV commit/rollback contract)
  verification pricing  engine.py:205-221
  answer phase          engine.py:538-560
  run_vanilla           engine.py:563-712
  validate_trajectory   engine.py:715-754

Comparisons against enums use ``==`` (the enums are ``str`` enums) rather than
identity, so results produced with the reference's own type objects are
accepted too; error classes are matched by name for the same reason.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Any

from .contract import Backend, FinishReason, GenerationRequest, VerificationRequest
from .contract import count_new_prompt_tokens
from .domain import (
    END_THINK_MARKER,
    VERIFY_HEAD_TOKENS,
    VERIFY_TAIL_TOKENS,
    BackendRole,
    Decision,
    EngineConfig,
    LatencyBreakdown,
    Phase,
    ReasoningStep,
    RunMetrics,
    Scheme,
    StepProducer,
    TrajectoryState,
    UtilityScore,
    count_tokens,
    decide_acceptance,
    render_generation_prompt,
    truncate_tokens,
)
from .pricing import derive_rng, rounds_latency, simulate_regen_rounds

ANSWER_MAX_TOKENS = 256


class StepAction(str, Enum):
    ACCEPTED_SPECULATION = "AcceptedSpeculation"
    REJECTED_THEN_REGENERATED = "RejectedThenRegenerated"
    FORCED_BASE = "ForcedBase"


@dataclass(frozen=True)
class StepOutcome:
    step: ReasoningStep
    action: StepAction

    def __post_init__(self) -> None:
        spec_kept = self.step.producer == StepProducer.SPECULATOR and self.step.accepted
        if spec_kept != (self.action == StepAction.ACCEPTED_SPECULATION):
            raise ValueError("action AcceptedSpeculation must match the step producer")

    def trace_record(self) -> dict:
        s = self.step
        return {
            "kind": "step",
            "index": s.index,
            "producer": s.producer.value,
            "score": s.score.value if s.score is not None else None,
            "action": self.action.value,
            "token_count": s.token_count,
            "speculate_s": s.latency.speculate_s,
            "verify_s": s.latency.verify_s,
            "fallback_s": s.latency.fallback_s,
        }


@dataclass
class TrajectoryResult:
    state: TrajectoryState
    outcomes: list[StepOutcome]
    metrics: RunMetrics
    rejected_steps: list[ReasoningStep]
    answer_latency_s: float
    trace: list[dict] = field(default_factory=list)


def force_first_n(config: EngineConfig, step_index: int) -> bool:
    return step_index < config.force_first_n


@dataclass(frozen=True)
class SegmentedStep:
    text: str
    end_think: bool
    truncated: bool


def segment_step(text: str, config: EngineConfig) -> SegmentedStep:
    """Cut one step off the front of ``text``: at ``</think>`` (marker
    dropped), at the earliest stop marker (kept, plus any directly following
    newlines), else at ``max_step_tokens`` whitespace units."""
    think_at = text.find(END_THINK_MARKER)
    cut_at, cut_end = -1, -1
    for marker in config.step_stop_markers:
        pos = text.find(marker)
        if pos >= 0 and (cut_at < 0 or pos < cut_at):
            cut_at, cut_end = pos, pos + len(marker)
    if think_at >= 0 and (cut_at < 0 or think_at < cut_at):
        return SegmentedStep(text[:think_at], True, False)
    if cut_at >= 0:
        n = len(text)
        while cut_end < n and text[cut_end] == "\n":
            cut_end += 1
        return SegmentedStep(text[:cut_end], False, False)
    if count_tokens(text) > config.max_step_tokens:
        return SegmentedStep(truncate_tokens(text, config.max_step_tokens), False, True)
    return SegmentedStep(text, False, False)


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

def _is_backend_error(exc: BaseException) -> bool:
    return any(k.__name__ == "BackendError" for k in type(exc).__mro__)


def _is_parse_failure(exc: BaseException) -> bool:
    return type(exc).__name__ == "ScoreParseFailure" or any(
        k.__name__ == "ScoreParseFailure" for k in type(exc).__mro__)


def _with_context(exc: BaseException, problem: str, step_index: int | None) -> BaseException:
    head = problem.splitlines()[0][:60] if problem else ""
    where = "" if step_index is None else f"step {step_index} of "
    return type(exc)(f"{where}problem {head!r}: {exc}")


@dataclass(frozen=True)
class _Piece:
    text: str
    token_count: int
    end_think: bool
    truncated: bool


def _generate_piece(backend: Backend, request: GenerationRequest, config: EngineConfig):
    """Call the backend and segment its text (engine.py:149-158)."""
    result = backend.generate_step(request)
    seg = segment_step(result.text, config)
    tokens = result.token_count if seg.text == result.text else backend.count_tokens(seg.text)
    return result, _Piece(
        text=seg.text,
        token_count=tokens,
        end_think=seg.end_think or result.finish_reason == FinishReason.END_THINK,
        truncated=seg.truncated or result.finish_reason == FinishReason.LENGTH,
    )


class PrefixLedger:
    """Logical prefix-cache streams ("small-gen", "base-gen", "base-verify").

    A stream remembers the longest content served; generated text extends a
    stream only when retained.  This is the commit/rollback contract that the
    B200 backend realises physically with KV pages (engine.py:161-186).
    """

    def __init__(self) -> None:
        self._streams: dict[str, str] = {}

    def seen(self, stream: str) -> bool:
        return stream in self._streams

    def charge(self, stream: str, content: str, backend: Backend) -> int:
        prev = self._streams.get(stream, "")
        fresh = count_new_prompt_tokens(prev, content, backend)
        if len(content) > len(prev):
            self._streams[stream] = content
        return fresh

    def extend(self, stream: str, content: str) -> None:
        if len(content) > len(self._streams.get(stream, "")):
            self._streams[stream] = content


def _gen_seconds(ledger: PrefixLedger, stream: str, backend: Backend, prompt: str,
                 result) -> float:
    if not backend.simulated:
        return result.measured_latency_s
    fresh = ledger.charge(stream, prompt, backend)
    return fresh / backend.profile.prefill_tokens_per_s + result.measured_latency_s


def _verify_seconds(ledger: PrefixLedger, base: Backend, problem: str, cot: str,
                    candidate_tokens: int) -> float:
    first = not ledger.seen("base-verify")
    fresh = ledger.charge("base-verify", problem + "\n" + cot, base)
    overhead = VERIFY_TAIL_TOKENS + (VERIFY_HEAD_TOKENS if first else 0)
    rate = base.profile.prefill_tokens_per_s
    return (fresh + candidate_tokens + overhead) / rate + base.profile.decode_s_per_token


def _fit_budget(piece: _Piece, remaining: int) -> tuple[str, int, bool]:
    if piece.token_count > remaining:
        return truncate_tokens(piece.text, remaining), remaining, True
    return piece.text, piece.token_count, False


def _step_request(prompt: str, config: EngineConfig) -> GenerationRequest:
    return GenerationRequest(prompt=prompt, max_tokens=config.max_step_tokens,
                             temperature=config.temperature,
                             stop=config.step_stop_markers, seed_hint=config.seed)


def _answer_request(prompt: str, config: EngineConfig) -> GenerationRequest:
    return GenerationRequest(prompt=prompt, max_tokens=ANSWER_MAX_TOKENS,
                             temperature=config.temperature, seed_hint=config.seed)


def _score(base: Backend, request: VerificationRequest) -> tuple[UtilityScore | None, float | None]:
    """Score; a parse failure is (None, ...) = Reject.  Seconds are measured
    for real backends and None for simulated ones (priced by the ledger)."""
    t0 = None if base.simulated else time.monotonic()
    try:
        score = base.score_step(request)
    except Exception as exc:  # noqa: BLE001 - re-raised unless a parse failure
        if not _is_parse_failure(exc):
            raise
        score = None
    return score, (None if t0 is None else time.monotonic() - t0)


# --------------------------------------------------------------------------
# SpecReason trajectory
# --------------------------------------------------------------------------

class _Run:
    """Mutable bookkeeping for one trajectory (single owner)."""

    def __init__(self, config: EngineConfig, problem: str) -> None:
        self.config = config
        self.state = TrajectoryState(problem=problem, budget=config.token_budget)
        self.ledger = PrefixLedger()
        self.outcomes: list[StepOutcome] = []
        self.rejected: list[ReasoningStep] = []
        self.trace: list[dict] = []
        self.index = 0
        self.carried = 0.0      # latency of a final no-text end-think, charged to the answer
        self.exhausted = False  # thinking ended on the budget

    def retain(self, text: str, tokens: int, producer: StepProducer,
               score: UtilityScore | None, latency: LatencyBreakdown,
               action: StepAction) -> None:
        step = ReasoningStep(index=self.index, text=text, token_count=tokens,
                             producer=producer, score=score, accepted=True,
                             latency=latency)
        outcome = StepOutcome(step, action)
        self.state.retained_steps.append(step)
        self.state.thinking_tokens_used += tokens
        self.outcomes.append(outcome)
        self.trace.append(outcome.trace_record())

    def end_thinking(self) -> None:
        self.state.phase = Phase.ANSWERING


def run_trajectory(config: EngineConfig, problem: str, small: Backend,
                   base: Backend) -> TrajectoryResult:
    """One full speculate / verify / fallback trajectory plus the answer."""
    if small.profile.role != BackendRole.SMALL:
        raise ValueError(f"small backend has role {small.profile.role.value}")
    if base.profile.role != BackendRole.BASE:
        raise ValueError(f"base backend has role {base.profile.role.value}")

    run = _Run(config, problem)
    try:
        answer_latency, exhausted = _think(run, small, base)
        answer_latency += _answer(run, base)
    except Exception as exc:
        if not _is_backend_error(exc):
            raise
        raise _with_context(exc, problem, len(run.state.retained_steps)) from exc

    kept = run.state.retained_steps
    n_spec = sum(1 for s in kept if s.producer == StepProducer.SPECULATOR)
    metrics = RunMetrics(
        latency_s=sum(s.latency.total_s for s in kept) + answer_latency,
        thinking_tokens=run.state.thinking_tokens_used,
        accepted_fraction=(n_spec / len(kept)) if kept else None,
        rejected_count=len(run.rejected),
        correct=False,
        scheme=Scheme.SPEC_REASON_DECODE if config.hierarchical else Scheme.SPEC_REASON,
        budget_exhausted=exhausted,
    )
    return TrajectoryResult(state=run.state, outcomes=run.outcomes, metrics=metrics,
                            rejected_steps=run.rejected, answer_latency_s=answer_latency,
                            trace=run.trace)


class SpecReasonSession:
    """Step-granular SpecReason trajectory (the same loop as
    ``run_trajectory``): ``step()`` runs one draft -> score -> accept / fall
    back iteration and returns the retained ``StepOutcome`` (None once
    thinking has ended); ``finish()`` generates the answer and returns the
    ``TrajectoryResult``.  Used by the benchmark to time individual steps."""

    def __init__(self, config: EngineConfig, problem: str, small: Backend, base: Backend) -> None:
        if small.profile.role != BackendRole.SMALL or base.profile.role != BackendRole.BASE:
            raise ValueError("small/base backends have the wrong roles")
        self.small, self.base = small, base
        self.run = _Run(config, problem)

    @property
    def thinking(self) -> bool:
        return self.run.state.phase == Phase.THINKING

    def step(self) -> StepOutcome | None:
        n = len(self.run.outcomes)
        try:
            _think_step(self.run, self.small, self.base)
        except Exception as exc:
            if not _is_backend_error(exc):
                raise
            raise _with_context(exc, self.run.state.problem, len(self.run.state.retained_steps)) from exc
        return self.run.outcomes[-1] if len(self.run.outcomes) > n else None

    def finish(self) -> TrajectoryResult:
        run = self.run
        while self.step() is not None or self.thinking:
            pass
        answer_latency = run.carried + _answer(run, self.base)
        kept = run.state.retained_steps
        n_spec = sum(1 for s in kept if s.producer == StepProducer.SPECULATOR)
        metrics = RunMetrics(
            latency_s=sum(s.latency.total_s for s in kept) + answer_latency,
            thinking_tokens=run.state.thinking_tokens_used,
            accepted_fraction=(n_spec / len(kept)) if kept else None,
            rejected_count=len(run.rejected), correct=False,
            scheme=Scheme.SPEC_REASON_DECODE if run.config.hierarchical else Scheme.SPEC_REASON,
            budget_exhausted=run.exhausted)
        return TrajectoryResult(state=run.state, outcomes=run.outcomes, metrics=metrics,
                                rejected_steps=run.rejected, answer_latency_s=answer_latency,
                                trace=run.trace)


def _regen_seconds(run: _Run, small: Backend, base: Backend, prompt: str, result) -> float:
    """Fallback cost; simulated + hierarchical runs price token-level rounds."""
    if not base.simulated:
        return result.measured_latency_s
    prefill_s = run.ledger.charge("base-gen", prompt, base) / base.profile.prefill_tokens_per_s
    agreement = getattr(base, "token_agreement_prob", None)
    if run.config.hierarchical and agreement is not None:
        rng = derive_rng("regen-rounds", base.profile.name, run.config.seed, run.index)
        rounds = simulate_regen_rounds(result.token_count, run.config.draft_length,
                                       agreement, rng)
        run.trace.append({"kind": "rounds", "step_index": run.index, "rounds": rounds})
        return prefill_s + rounds_latency(rounds, small.profile, base.profile)
    return prefill_s + result.measured_latency_s


def _think(run: _Run, small: Backend, base: Backend) -> tuple[float, bool]:
    """Thinking phase; returns (latency charged to the answer, budget hit)."""
    while _think_step(run, small, base):
        pass
    return run.carried, run.exhausted


def _think_step(run: _Run, small: Backend, base: Backend) -> bool:
    """One iteration of the thinking loop (engine.py:373-519); False once
    thinking has ended."""
    config, state = run.config, run.state
    if state.phase != Phase.THINKING:
        return False
    problem = state.problem
    remaining = state.budget - state.thinking_tokens_used
    if remaining <= 0:
        run.end_thinking()
        run.exhausted = True
        return False
    cot = state.cot_text()
    prompt = render_generation_prompt(problem, cot)
    request = _step_request(prompt, config)

    if force_first_n(config, run.index):
        res, piece = _generate_piece(base, request, config)
        secs = _gen_seconds(run.ledger, "base-gen", base, prompt, res)
        if piece.end_think and not piece.text:
            run.carried += secs
            run.end_thinking()
            return False
        text, tokens, hit = _fit_budget(piece, remaining)
        run.ledger.extend("base-gen", prompt + text)
        run.retain(text, tokens, StepProducer.BASE_FORCED, None,
                   LatencyBreakdown(fallback_s=secs), StepAction.FORCED_BASE)
        return _after_retain(run, hit, piece.end_think)

    cand_res, cand = _generate_piece(small, request, config)
    spec_s = _gen_seconds(run.ledger, "small-gen", small, prompt, cand_res)

    if cand.end_think and not cand.text:
        # the draft proposes to stop thinking: the base confirms or continues
        conf_res, conf = _generate_piece(base, request, config)
        conf_s = _gen_seconds(run.ledger, "base-gen", base, prompt, conf_res)
        if conf.end_think and not conf.text:
            run.carried += spec_s + conf_s
            run.end_thinking()
            return False
        text, tokens, hit = _fit_budget(conf, remaining)
        run.ledger.extend("base-gen", prompt + text)
        run.retain(text, tokens, StepProducer.BASE, None,
                   LatencyBreakdown(speculate_s=spec_s, fallback_s=conf_s),
                   StepAction.REJECTED_THEN_REGENERATED)
        return _after_retain(run, hit, conf.end_think)

    score, measured = _score(base, VerificationRequest(problem=problem, cot_prefix=cot,
                                                       candidate_step=cand.text))
    verify_s = (measured if measured is not None
                else _verify_seconds(run.ledger, base, problem, cot, cand.token_count))
    accepted = score is not None and decide_acceptance(score, config.threshold) == Decision.ACCEPT

    if accepted:
        text, tokens, hit = _fit_budget(cand, remaining)
        if small.simulated:
            run.ledger.extend("small-gen", prompt + text)
        run.retain(text, tokens, StepProducer.SPECULATOR, score,
                   LatencyBreakdown(speculate_s=spec_s, verify_s=verify_s),
                   StepAction.ACCEPTED_SPECULATION)
        return _after_retain(run, hit, cand.end_think)

    # Reject: audit copy, then the base regenerates from the same prefix
    run.rejected.append(ReasoningStep(
        index=run.index, text=cand.text, token_count=cand.token_count,
        producer=StepProducer.SPECULATOR, score=score, accepted=False,
        latency=LatencyBreakdown(speculate_s=spec_s, verify_s=verify_s)))
    regen_res, regen = _generate_piece(base, request, config)
    fb_s = _regen_seconds(run, small, base, prompt, regen_res)
    if regen.end_think and not regen.text:
        run.carried += spec_s + verify_s + fb_s
        run.end_thinking()
        return False
    text, tokens, hit = _fit_budget(regen, remaining)
    run.ledger.extend("base-gen", prompt + text)
    run.retain(text, tokens, StepProducer.BASE, None,
               LatencyBreakdown(speculate_s=spec_s, verify_s=verify_s, fallback_s=fb_s),
               StepAction.REJECTED_THEN_REGENERATED)
    run.trace[-1]["rejected_token_count"] = cand.token_count
    run.trace[-1]["rejected_score"] = score.value if score is not None else None
    return _after_retain(run, hit, regen.end_think)


def _after_retain(run: _Run, hit_budget: bool, end_think: bool) -> bool:
    """Advance the step index; end thinking on budget or end-think.  Returns
    whether thinking continues."""
    run.index += 1
    if hit_budget:
        run.exhausted = True
    if hit_budget or end_think:
        run.end_thinking()
        return False
    return True


def _answer(run: _Run, base: Backend) -> float:
    """Answer phase: the base answers after ``</think>``; not budgeted."""
    state = run.state
    state.phase = Phase.ANSWERING
    prompt = render_generation_prompt(state.problem, state.cot_text(), thinking_done=True)
    result = base.generate_step(_answer_request(prompt, run.config))
    secs = _gen_seconds(run.ledger, "base-gen", base, prompt, result)
    run.ledger.extend("base-gen", prompt + result.text)
    state.final_answer = result.text
    state.phase = Phase.DONE
    return secs


# --------------------------------------------------------------------------
# single-model baselines (BaseOnly / SmallOnly / SpecDecode pricing)
# --------------------------------------------------------------------------

def run_vanilla(config: EngineConfig, problem: str, backend: Backend,
                draft: Backend | None = None,
                token_speculative: bool = False) -> TrajectoryResult:
    """One backend produces every step and the answer, unscored."""
    try:
        return _vanilla(config, problem, backend, draft, token_speculative)
    except Exception as exc:
        if not _is_backend_error(exc):
            raise
        raise _with_context(exc, problem, None) from exc


def _vanilla(config: EngineConfig, problem: str, backend: Backend,
             draft: Backend | None, token_speculative: bool) -> TrajectoryResult:
    if token_speculative and draft is None:
        raise ValueError("token_speculative runs need a draft backend")
    is_small = backend.profile.role == BackendRole.SMALL
    if token_speculative:
        scheme = Scheme.SPEC_DECODE
    else:
        scheme = Scheme.SMALL_ONLY if is_small else Scheme.BASE_ONLY
    producer = StepProducer.SPECULATOR if is_small else StepProducer.BASE

    run = _Run(config, problem)
    state = run.state
    agreement = getattr(backend, "token_agreement_prob", None)
    priced_rounds = token_speculative and backend.simulated and agreement is not None
    tally = [0, 0]  # drafted, accepted

    def seconds(prompt: str, result) -> float:
        if not backend.simulated:
            return result.measured_latency_s
        prefill_s = run.ledger.charge("gen", prompt, backend) / backend.profile.prefill_tokens_per_s
        if priced_rounds and result.token_count > 0:
            rng = derive_rng("vanilla-rounds", backend.profile.name, config.seed, run.index)
            rounds = simulate_regen_rounds(result.token_count, config.draft_length,
                                           agreement, rng)
            run.trace.append({"kind": "rounds", "step_index": run.index, "rounds": rounds})
            tally[0] += sum(d for d, _ in rounds)
            tally[1] += sum(a for _, a in rounds)
            return prefill_s + rounds_latency(rounds, draft.profile, backend.profile)
        return prefill_s + result.measured_latency_s

    carried = 0.0
    exhausted = False
    while state.phase == Phase.THINKING:
        remaining = state.budget - state.thinking_tokens_used
        if remaining <= 0:
            exhausted = True
            run.end_thinking()
            break
        prompt = render_generation_prompt(problem, state.cot_text())
        res, piece = _generate_piece(backend, _step_request(prompt, config), config)
        secs = seconds(prompt, res)
        if piece.end_think and not piece.text:
            carried += secs
            run.end_thinking()
            break
        text, tokens, hit = _fit_budget(piece, remaining)
        run.ledger.extend("gen", prompt + text)
        if producer == StepProducer.SPECULATOR:
            lat, action = LatencyBreakdown(speculate_s=secs), StepAction.ACCEPTED_SPECULATION
        else:
            lat, action = LatencyBreakdown(fallback_s=secs), StepAction.FORCED_BASE
        run.retain(text, tokens, producer, None, lat, action)
        _after_retain(run, hit, piece.end_think)
        exhausted = exhausted or run.exhausted

    state.phase = Phase.ANSWERING
    prompt = render_generation_prompt(problem, state.cot_text(), thinking_done=True)
    result = backend.generate_step(_answer_request(prompt, config))
    run.index += 1
    carried += seconds(prompt, result)
    run.ledger.extend("gen", prompt + result.text)
    state.final_answer = result.text
    state.phase = Phase.DONE

    frac = None
    if scheme == Scheme.SPEC_DECODE and tally[0]:
        frac = tally[1] / tally[0]
    metrics = RunMetrics(
        latency_s=sum(s.latency.total_s for s in state.retained_steps) + carried,
        thinking_tokens=state.thinking_tokens_used,
        accepted_fraction=frac,
        rejected_count=0,
        correct=False,
        scheme=scheme,
        budget_exhausted=exhausted,
    )
    return TrajectoryResult(state=state, outcomes=run.outcomes, metrics=metrics,
                            rejected_steps=[], answer_latency_s=carried, trace=run.trace)


# --------------------------------------------------------------------------
# post-run invariants
# --------------------------------------------------------------------------

def validate_trajectory(result: TrajectoryResult, config: EngineConfig) -> None:
    """Raise ValueError on the first violated run invariant (engine.py:715-754)."""
    state = result.state
    kept = state.retained_steps
    if state.phase != Phase.DONE:
        raise ValueError(f"trajectory ended in phase {state.phase.value}")
    if state.thinking_tokens_used > state.budget:
        raise ValueError("thinking tokens exceed the budget")
    if state.thinking_tokens_used != sum(s.token_count for s in kept):
        raise ValueError("thinking_tokens_used disagrees with retained steps")
    if [o.step for o in result.outcomes] != kept:
        raise ValueError("outcome ordering disagrees with retained steps")
    kept_ids = {id(s) for s in kept}
    for s in result.rejected_steps:
        if id(s) in kept_ids:
            raise ValueError("a rejected step appears in the retained list")
        if s.accepted:
            raise ValueError("rejected steps must have accepted=False")
    if any(not s.accepted for s in kept):
        raise ValueError("retained steps must have accepted=True")
    if result.metrics.scheme in (Scheme.SPEC_REASON, Scheme.SPEC_REASON_DECODE):
        if any(s.producer == StepProducer.SPECULATOR and s.score is None for s in kept):
            raise ValueError("retained speculator steps must carry a score")
        regens = sum(1 for o in result.outcomes
                     if o.action == StepAction.REJECTED_THEN_REGENERATED)
        if len(result.rejected_steps) > regens + 1:
            raise ValueError("more audit rejections than regeneration outcomes")
    expected = sum(s.latency.total_s for s in kept) + result.answer_latency_s
    if abs(expected - result.metrics.latency_s) > 1e-9:
        raise ValueError("latency total disagrees with step breakdowns plus answer")


def trace_signature(result: Any) -> dict:
    """Timing-free fingerprint of a trajectory (works on reference results
    too): what parity tests compare between implementations."""
    state = result.state
    return {
        "steps": [(s.index, s.text, s.token_count, str(getattr(s.producer, "value", s.producer)),
                   None if s.score is None else s.score.value) for s in state.retained_steps],
        "rejected": [(s.index, s.text, s.token_count,
                      None if s.score is None else s.score.value)
                     for s in result.rejected_steps],
        "actions": [str(getattr(o.action, "value", o.action)) for o in result.outcomes],
        "answer": state.final_answer,
        "thinking_tokens": state.thinking_tokens_used,
        "budget_exhausted": result.metrics.budget_exhausted,
    }
