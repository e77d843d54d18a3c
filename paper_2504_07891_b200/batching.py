"""Several SpecReason trajectories per GPU with batched device calls (SURVEY
§8f-2).

The reference runs independent trajectories concurrently by handing one
``Backend`` pair to a thread pool (``bench.py:264-266``); its backends must be
thread-safe (``base.py:80-81``).  ``BatchScheduler`` keeps that contract and
adds what a GPU needs to profit from it: each trajectory thread calls a proxy
backend, the proxy parks the request, and a dispatcher thread releases the
parked requests as batched device passes -- ``generate_steps`` (one weight
stream per token for every live sequence, continuously batched: a new
generation joins the running ones at the next token) and ``score_steps`` (one
prefill pass over every candidate step that is waiting).

Trajectory semantics do not change: each request still gets exactly the
result its backend's single-request call returns (up to flagged near-ties,
``tests/test_gpu_batch.py``), so every thread's trajectory is the one it
would have produced alone.
"""

from __future__ import annotations

import os
import threading
import time
from concurrent.futures import Future
from typing import Any, Callable, Sequence


class _Proxy:
    """Backend-API stand-in that routes calls through the scheduler."""

    def __init__(self, sched: "BatchScheduler", backend: Any) -> None:
        self._sched = sched
        self._backend = backend

    def __getattr__(self, name: str) -> Any:  # profile, simulated, types, ...
        return getattr(self._backend, name)

    def generate_step(self, request):
        return self._sched._submit(self._backend, "gen", request)

    def score_step(self, request):
        return self._sched._submit(self._backend, "score", request)


class BatchScheduler:
    """Dispatches the parked requests of ``n_clients`` trajectory threads.

    A batch is released when every active client is waiting (nothing more can
    arrive) or ``linger_s`` after its first request, whichever comes first.
    """

    def __init__(self, small: Any, base: Any, linger_s: float = 0.002) -> None:
        for b in (small, base):
            pool = getattr(b, "pool", None)
            if pool is None or not hasattr(b, "_lock") or not hasattr(b, "engine"):
                raise TypeError(f"{type(b).__name__} is not a device ModelBackend "
                                "(needs pool, _lock and engine)")
            if len(pool.streams) < 2:
                raise ValueError("a scheduled backend needs at least 2 KV streams "
                                 "(one stays free for scoring)")
        self.small = _Proxy(self, small)
        self.base = _Proxy(self, base)
        self.linger_s = linger_s
        self._cv = threading.Condition()
        self._pending: list[tuple[Any, str, Any, Future]] = []
        self._active = 0
        self._stop = False
        self.batches: list[int] = []  # sizes of the device passes issued
        self._inflight: list = []     # the batch being dispatched
        self._thread = threading.Thread(target=self._loop, name="batch-dispatch", daemon=True)
        self._thread.start()

    # -- clients ---------------------------------------------------------------
    def _submit(self, backend: Any, kind: str, request: Any):
        fut: Future = Future()
        with self._cv:
            if self._stop:
                raise RuntimeError("BatchScheduler is closed (or its dispatcher failed)")
            self._pending.append((backend, kind, request, fut))
            self._cv.notify_all()
        res = fut.result()
        if isinstance(res, BaseException):
            raise res
        return res

    def run(self, jobs: Sequence[Callable[[Any, Any], Any]]) -> list:
        """Run ``job(small_proxy, base_proxy)`` for every job on its own thread;
        returns their results (or raised exceptions) in order."""
        out: list[Any] = [None] * len(jobs)

        def worker(i: int, job) -> None:
            try:
                out[i] = job(self.small, self.base)
            except BaseException as exc:  # recorded, like run_sweep's failures
                out[i] = exc
            finally:
                with self._cv:
                    self._active -= 1
                    self._cv.notify_all()

        with self._cv:
            self._active += len(jobs)
        threads = [threading.Thread(target=worker, args=(i, j)) for i, j in enumerate(jobs)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        return out

    def clients(self, n: int) -> "BatchScheduler":
        """Declare ``n`` client threads that the caller runs itself (e.g. the
        reference's ``run_sweep(..., parallelism=n)`` thread pool handed
        ``self.small`` / ``self.base``): a batch is then released once all
        ``n`` wait.  Undeclare with ``clients(-n)``."""
        with self._cv:
            self._active += n
            self._cv.notify_all()
        return self

    def close(self) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify_all()
        self._thread.join()

    # -- dispatcher ------------------------------------------------------------
    # Continuous batching: generations are opened as their requests arrive and
    # every live generation of a backend advances one token per device pass
    # (``engine.step_batch``: new prompts and single-token feeds share the
    # pass); scoring requests that arrive meanwhile run between two steps as
    # one ``score_steps`` pass.
    def _loop(self) -> None:
        live: dict[int, tuple[Any, list]] = {}  # id(backend) -> (backend, open generations)
        try:
            self._dispatch(live)
        except BaseException as exc:  # never leave a client blocked on its future
            with self._cv:
                pending, self._pending = self._pending + self._inflight, []
                self._stop = True
            for it in pending:
                if not it[3].done():
                    it[3].set_result(exc)
            for backend, gens in live.values():
                for g in gens:
                    backend.gen_release(g)
                    if not g["fut"].done():
                        g["fut"].set_result(exc)
                gens.clear()

    def _dispatch(self, live: dict) -> None:
        while True:
            with self._cv:
                busy = any(gs for _, gs in live.values())
                if not busy:
                    while not self._pending and not self._stop:
                        self._cv.wait()
                    if self._stop and not self._pending:
                        return
                    deadline = time.monotonic() + self.linger_s
                    while len(self._pending) < self._active and not self._stop:
                        left = deadline - time.monotonic()
                        if left <= 0:
                            break
                        self._cv.wait(left)
                batch, self._pending = self._pending, []
                self._inflight = batch
            self._scores([it for it in batch if it[1] == "score"])
            deferred = self._admit([it for it in batch if it[1] == "gen"], live)
            if deferred:
                with self._cv:
                    self._pending = deferred + self._pending
            busy_backends = sum(1 for _, gs in live.values() if gs)
            for backend, gens in live.values():
                if gens:
                    self._step(backend, gens, shared=busy_backends > 1)

    def _scores(self, items) -> None:
        groups: dict[int, list] = {}
        for it in items:
            groups.setdefault(id(it[0]), []).append(it)
        for chunk_all in groups.values():
            backend = chunk_all[0][0]
            cap = max(1, len(backend.pool.streams) - len(backend.pool.busy))  # free KV streams
            for i in range(0, len(chunk_all), cap):
                chunk = chunk_all[i:i + cap]
                reqs = [it[2] for it in chunk]
                try:
                    res = ([backend.score_step(reqs[0])] if len(reqs) == 1
                           else backend.score_steps(reqs))
                except BaseException as exc:
                    res = [exc] * len(chunk)
                self.batches.append(len(chunk))
                for it, r in zip(chunk, res):
                    it[3].set_result(r)

    def _admit(self, items, live) -> list:
        """Open generations for new requests; those that find no free KV
        stream wait for the next round."""
        deferred = []
        for backend, kind, req, fut in items:
            _, gens = live.setdefault(id(backend), (backend, []))
            if len(backend.pool.busy) >= len(backend.pool.streams) - 1:  # keep one for scoring
                deferred.append((backend, kind, req, fut))
                continue
            try:
                with backend._lock:
                    g = backend.gen_open(req, exclude=[x["stream"] for x in gens])
            except BaseException as exc:
                fut.set_result(exc)
                continue
            g["fut"] = fut
            gens.append(g)
        return deferred

    # a lone generation runs `solo_tokens` at a time on the single-stream
    # decode path (the persistent kernel) instead of one-token batched passes;
    # `solo_tokens_shared` when the other backend has live generations too, so
    # a long base chunk does not stall the drafts
    solo_tokens = 16
    solo_tokens_shared = int(os.environ.get("SR_SOLO_SHARED", "4"))

    def _step(self, backend, gens: list, shared: bool = False) -> None:
        if len(gens) == 1 and hasattr(backend.engine, "generate"):
            return self._solo(backend, gens, self.solo_tokens_shared if shared else self.solo_tokens)
        try:
            with backend._lock:
                toks = backend.engine.step_batch([g["stream"] for g in gens],
                                                 [g["feed"] for g in gens],
                                                 room=max(g["max"] - len(g["gen"]) for g in gens))
        except BaseException as exc:
            err = exc
            if isinstance(exc, RuntimeError) and type(exc).__name__ == "NativeError":
                err = backend._device_error(exc)
            for g in gens:
                backend.gen_release(g)
                g["fut"].set_result(err)
            gens.clear()
            return
        self.batches.append(len(gens))
        keep = []
        for g, t in zip(gens, toks):
            g["gen"].append(t)
            if backend.gen_done(g):
                try:
                    g["fut"].set_result(backend.gen_close(g))
                except BaseException as exc:
                    g["fut"].set_result(exc)
            else:
                g["feed"] = [t]
                keep.append(g)
        gens[:] = keep

    def _solo(self, backend, gens: list, chunk: int) -> None:
        g = gens[0]
        n = min(chunk, g["max"] - len(g["gen"]))
        try:
            with backend._lock:
                # stop ids end the chunk exactly as they end a generation
                toks, _ = backend.engine.generate(g["stream"], g["feed"], n, g["stop"])
        except BaseException as exc:
            err = exc
            if isinstance(exc, RuntimeError) and type(exc).__name__ == "NativeError":
                err = backend._device_error(exc)
            backend.gen_release(g)
            g["fut"].set_result(err)
            gens.clear()
            return
        self.batches.append(1)
        g["gen"].extend(toks)
        if backend.gen_done(g):
            try:
                g["fut"].set_result(backend.gen_close(g))
            except BaseException as exc:
                g["fut"].set_result(exc)
            gens.clear()
        else:
            g["feed"] = [toks[-1]]
