"""Host half of a model backend: tokenisation, prefix-cache streams, results.

``ModelBackend`` implements the reference plugin API (``Backend``,
``backends/base.py:77-100``) on top of a *device engine* that owns the model
arithmetic.  Two engines exist:

* ``backend.NativeEngine`` -- the product: sm_100a kernels behind the C-ABI
  in ``include/specreason_b200.h``;
* ``oracle.ref_engine.RefEngine`` -- the CPU fp32 oracle (tests only).

Both see exactly the same calls, so a parity failure can only come from the
arithmetic.

Semantics reproduced here (reference = the HTTP backend, the only one in the
reference that talks to a real model):

* generation: greedy continuation of the prompt; stop after the first token
  whose text contains a request stop string (the string is kept, as the
  engine's ``segment_step`` expects, ``engine.py:114-136``), drop ``</think>``
  and report ``END_THINK`` (``http.py:140-143``), else ``LENGTH`` at
  ``max_tokens``; latency is measured wall clock (``http.py:126-128``);
* scoring: the verify template (``prompts.py:52-77``), one prefill pass, and
  the readout of ``extract_score`` over the top-10 of the last position
  (``http.py:154-174``, ``base.py:106-126``), computed on the device;
  "no digit" raises ``ScoreParseFailure`` (the engine rejects).

Prefix caching (the reference's ``_PrefixLedger`` streams, ``engine.py:161-186``)
is realised physically: each device stream holds the token ids whose K/V are
resident; a call reuses the stream with the longest common prefix, rolls it
back to that prefix (rejected candidates, re-tokenised text) and prefills
only the rest -- the commit.
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass
from types import SimpleNamespace
from typing import Any, Protocol, Sequence

from . import contract, domain
from .contract import Backend, GenerationRequest, VerificationRequest
from .domain import BackendProfile
from .vocab import CLASS_END_THINK, CLASS_MASKED, CLASS_STOP, Vocab

# finish codes shared with the device (include/specreason_b200.h)
FINISH_LENGTH = 0
FINISH_STOP = 1
FINISH_END_THINK = 2


def own_types() -> SimpleNamespace:
    return SimpleNamespace(GenerationResult=contract.GenerationResult,
                           FinishReason=contract.FinishReason,
                           UtilityScore=domain.UtilityScore,
                           ScoreParseFailure=contract.ScoreParseFailure,
                           BackendMisbehavior=contract.BackendMisbehavior,
                           TransportError=contract.TransportError,
                           BackendProfile=domain.BackendProfile,
                           BackendRole=domain.BackendRole,
                           render_verification_prompt=domain.render_verification_prompt)


def reference_types(stepspec: Any) -> SimpleNamespace:
    """Bind results to the reference package's own classes, so the backend
    can be handed straight to the reference's ``run_trajectory``."""
    import importlib

    base = importlib.import_module(stepspec.__name__ + ".backends.base")
    core = importlib.import_module(stepspec.__name__ + ".core")
    prompts = importlib.import_module(stepspec.__name__ + ".prompts")
    return SimpleNamespace(GenerationResult=base.GenerationResult,
                           FinishReason=base.FinishReason,
                           UtilityScore=core.UtilityScore,
                           ScoreParseFailure=base.ScoreParseFailure,
                           BackendMisbehavior=base.BackendMisbehavior,
                           TransportError=base.TransportError,
                           BackendProfile=core.BackendProfile,
                           BackendRole=core.BackendRole,
                           render_verification_prompt=prompts.render_verification_prompt)


# --------------------------------------------------------------------------
# prefix-cache streams
# --------------------------------------------------------------------------

def common_prefix(a: Sequence[int], b: Sequence[int]) -> int:
    """Longest common prefix length (C-speed slice compares + bisection)."""
    n = min(len(a), len(b))
    if a[:n] == b[:n]:
        return n
    lo, hi = 0, n  # a[:lo] == b[:lo], a[:hi] != b[:hi]
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if a[lo:mid] == b[lo:mid]:
            lo = mid
        else:
            hi = mid
    return lo


class Stream:
    """One device KV stream: ``ids[i]`` has resident K/V at position i."""

    def __init__(self, sid: int) -> None:
        self.sid = sid
        self.ids: list[int] = []
        self.stamp = 0
        self.handle: Any = None  # engine-private (page table, ...)


class StreamPool:
    """Fixed set of streams; a prompt goes to the stream sharing the longest
    prefix with it (least recently used when none shares anything)."""

    def __init__(self, n: int) -> None:
        self.streams = [Stream(i) for i in range(n)]
        self._clock = 0
        # streams held by open (continuously batched) generations: never handed out
        self.busy: set = set()

    def acquire(self, ids: Sequence[int], exclude=()) -> tuple[Stream, int]:
        best, best_len = None, -1
        for s in self.streams:
            if s in exclude or s in self.busy:
                continue
            l = common_prefix(s.ids, ids)
            if l > best_len or (l == best_len and best is not None and s.stamp > best.stamp):
                best, best_len = s, l
        if best is None or best_len == 0:
            free = [s for s in self.streams if s not in exclude and s not in self.busy]
            if not free:
                raise RuntimeError("every KV stream of this backend is in use")
            best = min(free, key=lambda s: s.stamp)
            best_len = 0
        self._clock += 1
        best.stamp = self._clock
        # at least one prompt token is always recomputed: its logits seed
        # decode (an empty prompt keeps nothing: never a negative length)
        return best, max(0, min(best_len, len(ids) - 1))


# --------------------------------------------------------------------------
# engine protocol
# --------------------------------------------------------------------------

@dataclass
class Readout:
    """Device verify readout (the 16-byte record of the C-ABI)."""

    score: int          # -1: no digit (parse failure)
    accept: bool
    flags: int
    margin: float       # |top digit - runner-up| logit gap (ambiguity probe)
    argmax: int


class DeviceEngine(Protocol):
    spec: Any

    def attach(self, stream: Stream) -> None: ...
    def truncate(self, stream: Stream, keep: int) -> None: ...
    def generate(self, stream: Stream, suffix: Sequence[int], max_new: int,
                 classes_key: tuple[str, ...]) -> tuple[list[int], int]: ...
    def score(self, stream: Stream, suffix: Sequence[int], threshold: int) -> Readout: ...


# --------------------------------------------------------------------------
# the backend
# --------------------------------------------------------------------------

class _PromptCache:
    """Incremental tokenisation: re-use ids of a recent prompt that is a
    whitespace-terminated prefix of the new one."""

    def __init__(self, vocab: Vocab, size: int = 8) -> None:
        self.vocab = vocab
        self.size = size
        self.items: list[tuple[str, list[int]]] = []

    def encode(self, text: str) -> list[int]:
        for prev, ids in self.items:
            if len(prev) <= len(text) and prev and prev[-1].isspace() and text.startswith(prev):
                out = ids + self.vocab.encode(text[len(prev):])
                break
        else:
            out = self.vocab.encode(text)
        if text and text[-1].isspace():
            self.items.insert(0, (text, out))
            del self.items[self.size:]
        return out


class ModelBackend(Backend):
    """``Backend`` over a device engine (see module docstring)."""

    simulated = False

    def __init__(self, engine: DeviceEngine, vocab: Vocab, profile: BackendProfile,
                 n_streams: int = 4, threshold: int = 7, types: SimpleNamespace | None = None,
                 record: bool = False) -> None:
        self.engine = engine
        self.vocab = vocab
        self.profile = profile
        self.types = types or own_types()
        self.threshold = threshold
        self.pool = StreamPool(n_streams)
        self.engine.busy = self.pool.busy  # never evicted for another stream
        for s in self.pool.streams:
            engine.attach(s)
        self._lock = threading.Lock()
        self._prompts = _PromptCache(vocab)
        self.record = record
        self.calls: list[dict] = []   # per-call trace (ids) for replay parity
        self.verify_template = "v1"   # "v2": prefix-sharing verification prompts
        # a scoring call also prefills the base's generation stream up to the
        # same CoT (all but its last prompt token) in the same device pass, so
        # a fallback or the next base generation feeds one token and starts in
        # the decode kernel instead of a prefill pass (SR_CATCHUP=0: off)
        self.catch_up = os.environ.get("SR_CATCHUP", "1") != "0"

    # -- token-level speculation (SpecReason+Decode) ----------
    def attach_speculator(self, draft: "ModelBackend", gamma: int = 5) -> None:
        """Decode this (base) backend's steps with `draft` proposing `gamma`
        tokens per round and one verify pass accepting the longest prefix the
        greedy base agrees with, plus the base's own next token (lossless for
        greedy decoding: ``speculative_decode``, specdecode.py:120-177)."""
        if draft.vocab.n_text != self.vocab.n_text:
            raise ValueError("speculator must share the vocabulary")
        self.speculator = draft
        self.spec_gamma = int(gamma)
        self.spec_stats = {"rounds": 0, "proposed": 0, "accepted": 0}

    def _generate_speculative(self, ids: list[int], max_tokens: int,
                              stop: tuple[str, ...]) -> tuple[list[int], int]:
        d = self.speculator
        classes = self.vocab.token_classes(stop, max(self.vocab.n_text, 16))
        stream, keep = self.pool.acquire(ids)
        self.engine.truncate(stream, keep)
        ctx = list(ids)
        out: list[int] = []
        finish = FINISH_LENGTH
        with d._lock:
            dstream, dkeep = d.pool.acquire(ids)
            d.engine.truncate(dstream, dkeep)
            while True:
                budget = max_tokens - len(out)
                gamma = min(self.spec_gamma, budget)
                drafts: list[int] = []
                if gamma > 1:  # the verify pass always adds one base token itself
                    drafts, _ = d.engine.generate(dstream, ctx[len(dstream.ids):], gamma - 1, stop)
                if len(stream.ids) < len(ctx) - 1:  # catch the base stream up first
                    self.engine.prefill(stream, ctx[len(stream.ids):-1])
                choices, _ = self.engine.verify_tokens(stream, [ctx[-1]] + drafts)
                k = 0
                while k < len(drafts) and choices[k] == drafts[k]:
                    k += 1
                new = drafts[:k] + [choices[k]]
                self.spec_stats["rounds"] += 1
                self.spec_stats["proposed"] += len(drafts)
                self.spec_stats["accepted"] += k
                done = False
                for t in new:
                    out.append(t)
                    ctx.append(t)
                    c = int(classes[t]) if t < len(classes) else CLASS_MASKED
                    if c == CLASS_END_THINK:
                        finish, done = FINISH_END_THINK, True
                    elif c == CLASS_STOP:
                        finish, done = FINISH_STOP, True
                    elif len(out) >= max_tokens:
                        done = True
                    if done:
                        break
                # roll both streams back to the committed context (KV of ctx[:-1])
                self.engine.truncate(stream, min(len(stream.ids), len(ctx) - 1))
                d.engine.truncate(dstream, min(common_prefix(dstream.ids, ctx), len(ctx) - 1))
                if done:
                    return out, finish

    def _device_error(self, exc: Exception):
        """Map a native failure onto the reference's error hierarchy
        (base.py:19-32): collectives (NCCL) -> TransportError, everything
        else on the device -> BackendMisbehavior; the engine then adds the
        "step N of problem" context (engine.py:269-273)."""
        T = self.types
        code = getattr(exc, "code", None)
        cls = T.TransportError if code == 1004 else T.BackendMisbehavior
        return cls(f"{self.profile.name}: {exc}")

    # -- API -------------------------------------------------------------
    def generate_step(self, request: GenerationRequest):
        try:
            return self._generate_step(request)
        except RuntimeError as exc:
            if type(exc).__name__ != "NativeError":
                raise
            raise self._device_error(exc) from exc

    def score_step(self, request: VerificationRequest):
        try:
            return self._score_step(request)
        except RuntimeError as exc:
            if type(exc).__name__ != "NativeError":
                raise
            raise self._device_error(exc) from exc

    # -- several requests in one device pass -----------------
    def _acquire_many(self, id_lists):
        if len(id_lists) > len(self.pool.streams) - len(self.pool.busy):
            raise ValueError(f"{len(id_lists)} requests need as many KV streams "
                             f"(this backend has {len(self.pool.streams)})")
        chosen, keeps = [], []
        for ids in id_lists:
            st, keep = self.pool.acquire(ids, exclude=chosen)
            self.engine.truncate(st, keep)
            chosen.append(st)
            keeps.append(keep)
        return chosen, keeps

    def _native(self, fn, *args):
        """Run ``fn`` mapping a native failure like the single-request
        calls do (``_device_error``)."""
        try:
            return fn(*args)
        except RuntimeError as exc:
            if type(exc).__name__ != "NativeError":
                raise
            raise self._device_error(exc) from exc

    def score_steps(self, requests: Sequence[VerificationRequest]) -> list:
        return self._native(self._score_steps, requests)

    def _score_steps(self, requests: Sequence[VerificationRequest]) -> list:
        """``score_step`` for several independent requests in one device pass
        (the engine's ``score_batch``).  Results come back in request order: a
        ``UtilityScore``, or the ``ScoreParseFailure`` that ``score_step`` would
        have raised for that request."""
        T = self.types
        if self.profile.role != T.BackendRole.BASE:
            raise ValueError(f"backend {self.profile.name} cannot score steps")
        render = (domain.render_verification_prompt_v2 if self.verify_template == "v2"
                  else T.render_verification_prompt)
        with self._lock:
            id_lists = [self._prompts.encode(render(r.problem, r.cot_prefix, r.candidate_step))
                        for r in requests]
            streams, keeps = self._acquire_many(id_lists)
            rs = self.engine.score_batch(streams, [ids[k:] for ids, k in zip(id_lists, keeps)],
                                         self.threshold)
        return [T.UtilityScore(r.score) if r.score >= 0 else
                T.ScoreParseFailure("no digit in the top-10 or the sampled token") for r in rs]

    # continuous batching (batching.BatchScheduler): a generation is opened,
    # stepped together with other streams' generations, and closed
    def gen_open(self, request: GenerationRequest, exclude=()) -> dict:
        if not request.prompt:
            raise ValueError("prompt must be non-empty")
        ids = self._prompts.encode(request.prompt)
        if not ids:
            raise ValueError("prompt must contain at least one token")
        stream, keep = self.pool.acquire(ids, exclude=exclude)
        self.engine.truncate(stream, keep)
        self.pool.busy.add(stream)
        n_rows = getattr(self.engine, "n_ids", None) or self.engine.spec.vocab_rows
        return {"stream": stream, "feed": ids[keep:], "gen": [], "max": request.max_tokens,
                "stop": tuple(request.stop),
                "classes": self.vocab.token_classes(tuple(request.stop), n_rows),
                "t0": time.monotonic()}

    def gen_done(self, g: dict) -> bool:
        return (g["gen"] and g["classes"][g["gen"][-1]] in (CLASS_STOP, CLASS_END_THINK)) \
            or len(g["gen"]) >= g["max"]

    def gen_release(self, g: dict) -> None:
        self.pool.busy.discard(g["stream"])

    def gen_close(self, g: dict):
        self.gen_release(g)
        T = self.types
        gen = g["gen"]
        finish = finish_of(gen, g["classes"])
        if finish == FINISH_END_THINK:
            text_ids, reason = gen[:-1], T.FinishReason.END_THINK
        elif finish == FINISH_STOP:
            text_ids, reason = gen, T.FinishReason.STOP
        else:
            text_ids, reason = gen, T.FinishReason.LENGTH
        text = self.vocab.render(text_ids)
        if not text and reason == T.FinishReason.STOP:
            raise T.BackendMisbehavior("empty text with finish_reason stop")
        return T.GenerationResult(text=text, token_count=len(text_ids), finish_reason=reason,
                                  measured_latency_s=time.monotonic() - g["t0"])

    def generate_steps(self, requests: Sequence[GenerationRequest]) -> list:
        return self._native(self._generate_steps, requests)

    def _generate_steps(self, requests: Sequence[GenerationRequest]) -> list:
        """``generate_step`` for several independent requests, decoded together
        (the engine's ``generate_batch``: one weight stream per token for all
        live requests).  Returns ``GenerationResult`` in request order."""
        T = self.types
        stops = {tuple(r.stop) for r in requests}
        if len(stops) != 1 or len({r.max_tokens for r in requests}) != 1:
            raise ValueError("a batched generation needs one stop list and one max_tokens")
        t0 = time.monotonic()
        with self._lock:
            id_lists = [self._prompts.encode(r.prompt) for r in requests]
            streams, keeps = self._acquire_many(id_lists)
            max_new = requests[0].max_tokens
            outs = self.engine.generate_batch(streams, [ids[k:] for ids, k in zip(id_lists, keeps)],
                                              max_new, stops.pop())
        res = []
        for gen, finish in outs:
            if finish == FINISH_END_THINK:
                text_ids, reason = gen[:-1], T.FinishReason.END_THINK
            elif finish == FINISH_STOP:
                text_ids, reason = gen, T.FinishReason.STOP
            else:
                text_ids, reason = gen, T.FinishReason.LENGTH
            res.append(T.GenerationResult(text=self.vocab.render(text_ids),
                                          token_count=len(text_ids), finish_reason=reason,
                                          measured_latency_s=time.monotonic() - t0))
        return res

    def _generate_step(self, request: GenerationRequest):
        if not request.prompt:
            raise ValueError("prompt must be non-empty")
        t0 = time.monotonic()
        with self._lock:
            ids = self._prompts.encode(request.prompt)
            if not ids:
                raise ValueError("prompt must contain at least one token")
            if getattr(self, "speculator", None) is not None:
                gen, finish = self._generate_speculative(ids, request.max_tokens,
                                                         tuple(request.stop))
                keep = len(ids)
            else:
                stream, keep = self.pool.acquire(ids)
                self.engine.truncate(stream, keep)
                gen, finish = self.engine.generate(stream, ids[keep:], request.max_tokens,
                                                   tuple(request.stop))
            if self.record:
                self.calls.append({"kind": "gen", "prompt_ids": ids, "gen_ids": list(gen),
                                   "margins": ([] if getattr(self, "speculator", None) is not None
                                               else list(getattr(self.engine, "last_margins", []))),
                                   "finish": finish, "stop": list(request.stop),
                                   "max_tokens": request.max_tokens, "fresh": len(ids) - keep,
                                   "seq": time.monotonic_ns()})
        T = self.types
        if finish == FINISH_END_THINK:
            text_ids, reason = gen[:-1], T.FinishReason.END_THINK
        elif finish == FINISH_STOP:
            text_ids, reason = gen, T.FinishReason.STOP
        else:
            text_ids, reason = gen, T.FinishReason.LENGTH
        text = self.vocab.render(text_ids)
        if not text and reason == T.FinishReason.STOP:
            raise T.BackendMisbehavior("empty text with finish_reason stop")
        return T.GenerationResult(text=text, token_count=len(text_ids), finish_reason=reason,
                                  measured_latency_s=time.monotonic() - t0)

    def _catch_up_plan(self, request, vstream, v_rows: int):
        """(stream, keep, ids) of the generation stream a scoring call extends
        in its own device pass, or None.  The generation prompt of the same CoT
        (``render_generation_prompt(problem, cot_prefix)``: what a fallback or
        the next base generation feeds) is cached up to its last token, on the
        stream with the longest common prefix other than the verify stream.
        Only when at least two rows are missing: with one, the generation
        already starts in the decode kernel (``sr_generate``'s one-token path),
        which keeps a base that generates every step (threshold 10) computing
        exactly what ``run_vanilla`` does.  Never on a trajectory's first step
        (empty CoT): ``run_vanilla``'s first generation prefills the whole
        prompt and takes its first token from that pass's LM head, so a
        threshold-10 fallback must do the same rather than start in the
        decode kernel."""
        if (not self.catch_up or self.verify_template != "v1" or len(self.pool.streams) < 2
                or not getattr(self.engine, "multi_span_passes", False)
                or not request.cot_prefix):
            return None
        gids = self._prompts.encode(domain.render_generation_prompt(request.problem,
                                                                    request.cot_prefix))
        if len(gids) < 3:
            return None
        gst, gkeep = self.pool.acquire(gids[:-1], exclude=(vstream,))
        n = len(gids) - 1 - gkeep
        if n < 2 or n + v_rows > self.engine.model.max_tokens:
            return None
        return gst, gkeep, gids

    def _score_step(self, request: VerificationRequest):
        T = self.types
        if self.profile.role != T.BackendRole.BASE:
            raise ValueError(f"backend {self.profile.name} cannot score steps")
        if self.verify_template == "v2":  # prefix-sharing (opt-in; §8f-3)
            prompt = domain.render_verification_prompt_v2(request.problem, request.cot_prefix,
                                                          request.candidate_step)
        else:
            prompt = T.render_verification_prompt(request.problem, request.cot_prefix,
                                                  request.candidate_step)
        with self._lock:
            ids = self._prompts.encode(prompt)
            stream, keep = self.pool.acquire(ids)
            self.engine.truncate(stream, keep)
            catch = self._catch_up_plan(request, stream, len(ids) - keep)
            if catch is None:
                r = self.engine.score(stream, ids[keep:], self.threshold)
            else:
                gst, gkeep, gids = catch
                self.engine.truncate(gst, gkeep)
                r = self.engine.score_batch([stream, gst], [ids[keep:], gids[gkeep:-1]],
                                            self.threshold)[0]
            if self.record:
                self.calls.append({"kind": "score", "prompt_ids": ids, "score": r.score,
                                   "accept": r.accept, "margin": r.margin,
                                   "argmax": r.argmax, "fresh": len(ids) - keep,
                                   "seq": time.monotonic_ns(),
                                   **({"catchup_start": catch[1],
                                       "catchup": len(catch[2]) - 1 - catch[1]} if catch else {})})
        if r.score < 0:
            raise T.ScoreParseFailure("no digit in the top-10 or the sampled token")
        return T.UtilityScore(r.score)


def finish_of(ids: Sequence[int], classes) -> int:
    """Finish code of a generated id run under a class table (host mirror of
    the device stop test, used by the CPU engine and by tests)."""
    if not ids:
        return FINISH_LENGTH
    c = int(classes[ids[-1]])
    if c == CLASS_END_THINK:
        return FINISH_END_THINK
    if c == CLASS_STOP:
        return FINISH_STOP
    return FINISH_LENGTH
