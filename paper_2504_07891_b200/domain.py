"""Value types, the judge rule, prompt layouts and the whitespace token model.

Host-side mirror of the reference ``stepspec`` domain layer so that a user of
the reference finds the same names with the same behaviour:

* scores / thresholds / acceptance  -> ``pkg/src/stepspec/core.py:63-93``
* step, trajectory, config, profile, metrics types -> ``core.py:96-369``
* prompt layouts and the token model -> ``pkg/src/stepspec/prompts.py:13-98``

Everything is a plain value type (frozen dataclasses, ``str`` enums with the
reference's literal values) so JSON produced by one implementation parses in
the other.  Only ``TrajectoryState`` is mutable and it has a single writer
(the driver loop that owns it).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from enum import Enum
from typing import Any

# --------------------------------------------------------------------------
# markers and enums (core.py:14-54)
# --------------------------------------------------------------------------

END_THINK_MARKER = "</think>"
THINK_OPEN_MARKER = "<think>"
MAX_UTILITY_SCORE = 9


class StepProducer(str, Enum):
    SPECULATOR = "Speculator"
    BASE = "Base"
    BASE_FORCED = "BaseForced"


class Phase(str, Enum):
    THINKING = "Thinking"
    ANSWERING = "Answering"
    DONE = "Done"


class Decision(str, Enum):
    ACCEPT = "Accept"
    REJECT = "Reject"


class BackendRole(str, Enum):
    SMALL = "Small"
    BASE = "Base"


class Scheme(str, Enum):
    BASE_ONLY = "BaseOnly"
    SMALL_ONLY = "SmallOnly"
    SPEC_DECODE = "SpecDecode"
    SPEC_REASON = "SpecReason"
    SPEC_REASON_DECODE = "SpecReasonDecode"


SPECULATIVE_SCHEMES = frozenset(
    (Scheme.SPEC_DECODE, Scheme.SPEC_REASON, Scheme.SPEC_REASON_DECODE)
)


def _strict_int(label: str, value: Any) -> int:
    # bool is an int subclass; the reference rejects it (core.py:57-60)
    if type(value) is bool or not isinstance(value, int):
        raise TypeError(f"{label} must be an int, got {type(value).__name__}")
    return value


# --------------------------------------------------------------------------
# judge rule (core.py:63-93)
# --------------------------------------------------------------------------

@dataclass(frozen=True, order=True)
class UtilityScore:
    """Single-digit judgment 0..9 of a candidate step."""

    value: int

    def __post_init__(self) -> None:
        v = _strict_int("score", self.value)
        if v < 0 or v > MAX_UTILITY_SCORE:
            raise ValueError(f"utility score must be in [0, 9], got {v}")


@dataclass(frozen=True, order=True)
class AcceptanceThreshold:
    """Minimum accepted score; 0 accepts all, 10 rejects all (pure fallback)."""

    value: int

    def __post_init__(self) -> None:
        v = _strict_int("threshold", self.value)
        if v < 0 or v > MAX_UTILITY_SCORE + 1:
            raise ValueError(f"threshold must be in [0, 10], got {v}")


def decide_acceptance(score: UtilityScore, threshold: AcceptanceThreshold) -> Decision:
    """score >= threshold accepts (boundary accepted), core.py:91-93."""
    if score.value >= threshold.value:
        return Decision.ACCEPT
    return Decision.REJECT


# --------------------------------------------------------------------------
# JSON helpers shared by the record types
# --------------------------------------------------------------------------

def _plain(value: Any) -> Any:
    if isinstance(value, Enum):
        return value.value
    if dataclasses.is_dataclass(value) and [f.name for f in dataclasses.fields(value)] == ["value"]:
        return value.value  # UtilityScore / AcceptanceThreshold (ours or the reference's)
    if isinstance(value, tuple):
        return list(value)
    if hasattr(value, "to_dict"):
        return value.to_dict()
    if isinstance(value, list):
        return [_plain(v) for v in value]
    return value


def _as_dict(obj: Any, names: tuple[str, ...]) -> dict[str, Any]:
    return {n: _plain(getattr(obj, n)) for n in names}


# --------------------------------------------------------------------------
# latency, steps, trajectory (core.py:96-222)
# --------------------------------------------------------------------------

_LATENCY_KEYS = ("speculate_s", "verify_s", "fallback_s")


@dataclass(frozen=True)
class LatencyBreakdown:
    """Seconds charged to one step slot: draft, verify, base generation."""

    speculate_s: float = 0.0
    verify_s: float = 0.0
    fallback_s: float = 0.0

    def __post_init__(self) -> None:
        for key in _LATENCY_KEYS:
            if getattr(self, key) < 0:
                raise ValueError(f"{key} must be >= 0")

    @property
    def total_s(self) -> float:
        return self.speculate_s + self.verify_s + self.fallback_s

    def to_dict(self) -> dict[str, float]:
        return _as_dict(self, _LATENCY_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "LatencyBreakdown":
        return cls(**{k: data[k] for k in _LATENCY_KEYS})


def total_latency(step: "ReasoningStep") -> float:
    return step.latency.total_s


_STEP_KEYS = ("index", "text", "token_count", "producer", "score", "accepted", "latency")


@dataclass(frozen=True)
class ReasoningStep:
    index: int
    text: str
    token_count: int
    producer: StepProducer
    score: UtilityScore | None
    accepted: bool
    latency: LatencyBreakdown

    def __post_init__(self) -> None:
        if self.index < 0:
            raise ValueError("step index must be >= 0")
        if self.token_count < 0:
            raise ValueError("token_count must be >= 0")
        if self.text and self.token_count == 0:
            raise ValueError("non-empty step text must count at least one token")
        if self.score is not None and self.producer is not StepProducer.SPECULATOR:
            raise ValueError("only speculator-produced steps carry a score")

    def to_dict(self) -> dict[str, Any]:
        return _as_dict(self, _STEP_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "ReasoningStep":
        raw_score = data["score"]
        return cls(
            index=data["index"],
            text=data["text"],
            token_count=data["token_count"],
            producer=StepProducer(data["producer"]),
            score=UtilityScore(raw_score) if raw_score is not None else None,
            accepted=data["accepted"],
            latency=LatencyBreakdown.from_dict(data["latency"]),
        )


_STATE_KEYS = ("problem", "retained_steps", "thinking_tokens_used", "phase", "budget",
               "final_answer")


@dataclass
class TrajectoryState:
    """Retained chain of steps for one problem (single writer)."""

    problem: str
    retained_steps: list[ReasoningStep] = field(default_factory=list)
    thinking_tokens_used: int = 0
    phase: Phase = Phase.THINKING
    budget: int = 8192
    final_answer: str | None = None

    def cot_text(self) -> str:
        return "".join(s.text for s in self.retained_steps)

    def to_dict(self) -> dict[str, Any]:
        return _as_dict(self, _STATE_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "TrajectoryState":
        return cls(
            problem=data["problem"],
            retained_steps=[ReasoningStep.from_dict(s) for s in data["retained_steps"]],
            thinking_tokens_used=data["thinking_tokens_used"],
            phase=Phase(data["phase"]),
            budget=data["budget"],
            final_answer=data["final_answer"],
        )


# --------------------------------------------------------------------------
# engine config, backend profile, run metrics (core.py:225-369)
# --------------------------------------------------------------------------

DEFAULT_STEP_STOP_MARKERS: tuple[str, ...] = ("\n\n", ".\n", "!\n", "?\n")

_CONFIG_KEYS = ("threshold", "force_first_n", "token_budget", "temperature", "draft_length",
                "hierarchical", "seed", "max_step_tokens", "step_stop_markers")


@dataclass(frozen=True)
class EngineConfig:
    """Run knobs (defaults: threshold 7, budget 8192, temperature 0.6)."""

    threshold: AcceptanceThreshold = AcceptanceThreshold(7)
    force_first_n: int = 0
    token_budget: int = 8192
    temperature: float = 0.6
    draft_length: int = 5
    hierarchical: bool = False
    seed: int = 0
    max_step_tokens: int = 256
    step_stop_markers: tuple[str, ...] = DEFAULT_STEP_STOP_MARKERS

    def __post_init__(self) -> None:
        checks = (
            (self.force_first_n >= 0, "force_first_n must be >= 0"),
            (self.token_budget >= 1, "token_budget must be >= 1"),
            (self.temperature >= 0, "temperature must be >= 0"),
            (self.draft_length >= 1, "draft_length must be >= 1"),
            (self.max_step_tokens >= 1, "max_step_tokens must be >= 1"),
        )
        for ok, message in checks:
            if not ok:
                raise ValueError(message)
        if not isinstance(self.step_stop_markers, tuple):
            object.__setattr__(self, "step_stop_markers", tuple(self.step_stop_markers))

    def to_dict(self) -> dict[str, Any]:
        return _as_dict(self, _CONFIG_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "EngineConfig":
        kwargs = {k: data[k] for k in _CONFIG_KEYS}
        kwargs["threshold"] = AcceptanceThreshold(kwargs["threshold"])
        kwargs["step_stop_markers"] = tuple(kwargs["step_stop_markers"])
        return cls(**kwargs)


_PROFILE_KEYS = ("name", "role", "decode_s_per_token", "prefill_tokens_per_s")


@dataclass(frozen=True)
class BackendProfile:
    """Backend identity plus the two-parameter latency model."""

    name: str
    role: BackendRole
    decode_s_per_token: float
    prefill_tokens_per_s: float

    def __post_init__(self) -> None:
        if not self.decode_s_per_token > 0:
            raise ValueError("decode_s_per_token must be > 0")
        if not self.prefill_tokens_per_s > 0:
            raise ValueError("prefill_tokens_per_s must be > 0")

    def to_dict(self) -> dict[str, Any]:
        return _as_dict(self, _PROFILE_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "BackendProfile":
        kwargs = {k: data[k] for k in _PROFILE_KEYS}
        kwargs["role"] = BackendRole(kwargs["role"])
        return cls(**kwargs)


_METRIC_KEYS = ("latency_s", "thinking_tokens", "accepted_fraction", "rejected_count",
                "correct", "scheme", "budget_exhausted")


@dataclass(frozen=True)
class RunMetrics:
    latency_s: float
    thinking_tokens: int
    accepted_fraction: float | None
    rejected_count: int
    correct: bool
    scheme: Scheme
    budget_exhausted: bool

    def __post_init__(self) -> None:
        for key in ("latency_s", "thinking_tokens", "rejected_count"):
            if getattr(self, key) < 0:
                raise ValueError(f"{key} must be >= 0")
        frac = self.accepted_fraction
        if self.scheme not in SPECULATIVE_SCHEMES:
            if frac is not None:
                raise ValueError(
                    f"accepted_fraction is undefined for scheme {self.scheme.value}")
        elif frac is not None and not (0 <= frac <= 1):
            raise ValueError("accepted_fraction must be in [0, 1]")

    def to_dict(self) -> dict[str, Any]:
        return _as_dict(self, _METRIC_KEYS)

    @classmethod
    def from_dict(cls, data: dict[str, Any]) -> "RunMetrics":
        kwargs = {k: data[k] for k in _METRIC_KEYS}
        kwargs["scheme"] = Scheme(kwargs["scheme"])
        return cls(**kwargs)


# --------------------------------------------------------------------------
# token model and prompt layouts (prompts.py:13-98)
# --------------------------------------------------------------------------

def count_tokens(text: str) -> int:
    """One token per whitespace-delimited unit (prompts.py:13-14)."""
    return len(text.split())


def truncate_tokens(text: str, max_tokens: int) -> str:
    """First ``max_tokens`` units, re-joined by single spaces when cut
    (prompts.py:17-24); text that already fits is returned untouched."""
    if max_tokens <= 0:
        return ""
    words = text.split()
    return text if len(words) <= max_tokens else " ".join(words[:max_tokens])


_THINK_OPENER = "\n" + THINK_OPEN_MARKER + "\n"


def render_generation_prompt(problem: str, cot: str, thinking_done: bool = False) -> str:
    """``problem \\n<think>\\n cot`` (+ ``</think>\\n`` for the answer)."""
    tail = END_THINK_MARKER + "\n" if thinking_done else ""
    return problem + _THINK_OPENER + cot + tail


def split_generation_prompt(prompt: str) -> tuple[str, str, bool]:
    """Inverse of :func:`render_generation_prompt` -> (problem, cot, answering)."""
    problem, sep, cot = prompt.partition(_THINK_OPENER)
    if not sep:
        problem, cot = prompt, ""
    answering = END_THINK_MARKER in cot
    if answering:
        cot = cot.partition(END_THINK_MARKER)[0]
    return problem, cot, answering


# The judge template is a versioned literal: its wording fixes the token
# layout of every verification prefill, so it must equal the reference's
# VERIFY_PROMPT_V1 (prompts.py:52-66) character for character.
VERIFY_PROMPT_VERSION = "v1"
VERIFY_PROMPT_V1 = (
    "You are grading one candidate step of a running solution.\n"
    "\n"
    "Problem:\n"
    "{problem}\n"
    "\n"
    "Reasoning so far:\n"
    "{cot_prefix}\n"
    "\n"
    "Candidate next step:\n"
    "{candidate_step}\n"
    "\n"
    "Judge only the candidate step. A high score means the step is correct,\n"
    "relevant, and moves the reasoning forward; a low score means it is wrong,\n"
    "redundant, or off-track.\n"
    "Respond with a single digit 0-9:"
)


# Prefix-sharing verification template (not the reference's
# wording, so scores are not comparable with VERIFY_PROMPT_V1 and it is
# opt-in).  It starts with the generation prompt itself -- problem, the think
# marker, the CoT -- and appends the candidate as the next step, so the base
# model's generation stream already holds the K/V of everything but the
# candidate and the short tail, and an accepted candidate's K/V stays in place
# for the next step.  The last word is the same judge cue as V1's.
VERIFY_PROMPT_V2_TAIL = (
    "\n\nJudge only the last step above. A high score means the step is correct,\n"
    "relevant, and moves the reasoning forward; a low score means it is wrong,\n"
    "redundant, or off-track.\n"
    "Respond with a single digit 0-9:"
)


def render_verification_prompt_v2(problem: str, cot_prefix: str, candidate_step: str) -> str:
    return render_generation_prompt(problem, cot_prefix) + candidate_step + VERIFY_PROMPT_V2_TAIL


def render_verification_prompt(problem: str, cot_prefix: str, candidate_step: str,
                               template: str = VERIFY_PROMPT_V1) -> str:
    return template.format(problem=problem, cot_prefix=cot_prefix,
                           candidate_step=candidate_step)


def verification_sections(template: str = VERIFY_PROMPT_V1) -> tuple[str, str, str, str]:
    """(head, mid1, mid2, tail) around {problem}, {cot_prefix}, {candidate_step}."""
    pieces = []
    rest = template
    for slot in ("{problem}", "{cot_prefix}", "{candidate_step}"):
        before, _, rest = rest.partition(slot)
        pieces.append(before)
    pieces.append(rest)
    return tuple(pieces)  # type: ignore[return-value]


def verification_overhead_tokens(template: str = VERIFY_PROMPT_V1) -> tuple[int, int]:
    """(head+mid1 tokens, mid2+tail tokens) of template text."""
    head, mid1, mid2, tail = verification_sections(template)
    return count_tokens(head + " " + mid1), count_tokens(mid2 + " " + tail)


VERIFY_HEAD_TOKENS, VERIFY_TAIL_TOKENS = verification_overhead_tokens()


def replace(obj: Any, **changes: Any) -> Any:
    """``dataclasses.replace`` re-export (the engine/bench use it on configs)."""
    return dataclasses.replace(obj, **changes)
