"""Keyed seeds and the round-structure price model used by the driver.

Only *simulated* backends are priced through these functions; a real backend
(``B200Backend``) reports measured wall clock and never reaches them.  They
exist so the driver keeps the reference's accounting bit-for-bit when a
simulated backend is plugged in:

* ``derive_seed`` / ``derive_rng``  -> ``pkg/src/stepspec/seeding.py:19-33``
* ``trajectory_seed``               -> ``pkg/src/stepspec/bench.py:216-218``
* ``simulate_regen_rounds``         -> ``pkg/src/stepspec/specdecode.py:180-206``
* ``rounds_latency``                -> ``pkg/src/stepspec/specdecode.py:209-225``
"""

from __future__ import annotations

import hashlib
from typing import Any, Sequence

import numpy as np

from .domain import BackendProfile


def _key_digest(parts: tuple[Any, ...]) -> bytes:
    # blake2b-128 over repr()-encoded parts, each followed by a 0x1f separator
    h = hashlib.blake2b(digest_size=16)
    for part in parts:
        h.update(part if isinstance(part, bytes) else repr(part).encode("utf-8"))
        h.update(b"\x1f")
    return h.digest()


def derive_seed(*parts: Any) -> int:
    """Stable 64-bit seed: the first 8 digest bytes, big-endian."""
    return int.from_bytes(_key_digest(parts)[:8], "big")


def derive_rng(*parts: Any) -> np.random.Generator:
    """numpy PCG64 substream seeded by the full 128-bit digest."""
    return np.random.default_rng(int.from_bytes(_key_digest(parts), "big"))


def trajectory_seed(base_seed: int, problem_id: str, repeat: int) -> int:
    """Per-(problem, repeat) seed, independent of knob values and of how the
    problems are partitioned across GPUs."""
    return derive_seed("trajectory", base_seed, problem_id, repeat)


def simulate_regen_rounds(total_tokens: int, gamma: int, agreement_prob: float,
                          rng: np.random.Generator) -> list[tuple[int, int]]:
    """(drafted, accepted) per token-speculation round for a step of known
    length; every round appends accepted+1 tokens (at most what remains)."""
    if total_tokens < 0:
        raise ValueError("total_tokens must be >= 0")
    if gamma < 1:
        raise ValueError("gamma must be >= 1")
    if not 0 <= agreement_prob <= 1:
        raise ValueError("agreement_prob must be in [0, 1]")
    out: list[tuple[int, int]] = []
    left = total_tokens
    while left > 0:
        drafted = gamma if gamma < left else left
        hit = 0
        while hit < drafted and rng.random() < agreement_prob:
            hit += 1
        out.append((drafted, hit))
        left -= min(hit + 1, left)
    return out


def rounds_latency(rounds: Sequence[tuple[int, int]], draft_profile: BackendProfile,
                   target_profile: BackendProfile) -> float:
    """Draft decodes its drafted tokens, target prefills them plus one decode."""
    seconds = 0.0
    for drafted, _ in rounds:
        seconds += drafted * draft_profile.decode_s_per_token
        seconds += drafted / target_profile.prefill_tokens_per_s + target_profile.decode_s_per_token
    return seconds
