"""B200-measured ``BackendProfile``.

The reference calibrates its latency model with the ``profile`` CLI verb
(``cli.py:399-442``): two-point fits over ``generate_step`` calls against an
OpenAI-compatible server -- decode seconds per token from a 96- vs an 8-token
decode of one prompt, and prefill tokens per second from a 600- vs an 8-word
``"echo "`` prompt decoded for one token.  ``measure_profile`` runs the same
fits through a B200 backend's own ``generate_step``, so the numbers it returns
can be fed to the reference's simulator (``simlab.py:330-343`` defaults) or
stored with a sweep.  The same errors are raised for the same conditions.

Each fit point takes the fastest of ``reps`` repetitions (the reference takes a
single sample of a remote server; here the device is local and the minimum
removes host jitter).  Prefix caching is defeated by truncating the backend's
streams before every call, because the reference's server would re-prefill a
fresh request too (``http.py:121-152`` sends the whole prompt each time).
"""

from __future__ import annotations

from dataclasses import replace
from typing import Any

from . import contract
from .domain import BackendProfile

DECODE_PROMPT = "Count upward from one, separating numbers with spaces:"


def _fresh(backend: Any) -> None:
    for s in backend.pool.streams:
        backend.engine.truncate(s, 0)
        s.ids.clear()


def _timed(backend: Any, prompt: str, max_tokens: int, reps: int):
    best = None
    for _ in range(reps):
        _fresh(backend)
        r = backend.generate_step(contract.GenerationRequest(prompt=prompt, max_tokens=max_tokens))
        if best is None or r.measured_latency_s < best.measured_latency_s:
            best = r
    return best


def measure_profile(backend: Any, reps: int = 3) -> Any:
    """Return ``backend.profile`` with measured ``decode_s_per_token`` and
    ``prefill_tokens_per_s`` (same class as the backend's profile)."""
    short = _timed(backend, DECODE_PROMPT, 8, reps)
    long = _timed(backend, DECODE_PROMPT, 96, reps)
    if long.token_count <= short.token_count:
        raise RuntimeError("server did not decode more tokens at a larger max_tokens")
    decode_s = (long.measured_latency_s - short.measured_latency_s) / (
        long.token_count - short.token_count)
    if decode_s <= 0:
        raise RuntimeError("measured non-positive decode time; rerun on a quieter server")
    p_short = _timed(backend, "echo " * 8, 1, reps)
    p_long = _timed(backend, "echo " * 600, 1, reps)
    delta_t = p_long.measured_latency_s - p_short.measured_latency_s
    if delta_t <= 0:
        raise RuntimeError("measured non-positive prefill time; rerun on a quieter server")
    _fresh(backend)
    prof = backend.profile
    try:
        return replace(prof, decode_s_per_token=decode_s, prefill_tokens_per_s=(600 - 8) / delta_t)
    except TypeError:  # a profile class that is not a dataclass
        return type(prof)(name=prof.name, role=prof.role, decode_s_per_token=decode_s,
                          prefill_tokens_per_s=(600 - 8) / delta_t)


def profile_dict(p: Any) -> dict:
    """The profile fields the reference's config file holds (``cli.py``)."""
    role = getattr(p.role, "value", p.role)
    return {"name": p.name, "role": role, "decode_s_per_token": p.decode_s_per_token,
            "prefill_tokens_per_s": p.prefill_tokens_per_s}


__all__ = ["measure_profile", "profile_dict", "BackendProfile", "DECODE_PROMPT"]
