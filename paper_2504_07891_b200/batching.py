"""Several SpecReason trajectories per GPU with batched device calls (SURVEY
§8f-2).

The reference runs independent trajectories concurrently by handing one
``Backend`` pair to a thread pool (``bench.py:264-266``); its backends must be
thread-safe (``base.py:80-81``).  ``BatchScheduler`` keeps that contract and
adds what a GPU needs to profit from it: each trajectory thread calls a proxy
backend, the proxy parks the request, and a dispatcher thread releases the
parked requests as batched device passes -- ``generate_steps`` (one weight
stream per token for every live sequence) and ``score_steps`` (one prefill
pass over every candidate step).  Requests are grouped by (backend, kind,
stop list, max_tokens); a group larger than the backend's KV streams is split.

Trajectory semantics do not change: each request still gets exactly the
result its backend's single-request call returns (up to flagged near-ties,
``tests/test_gpu_batch.py``), so every thread's trajectory is the one it
would have produced alone.
"""

from __future__ import annotations

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
        self.small = _Proxy(self, small)
        self.base = _Proxy(self, base)
        self.linger_s = linger_s
        self._cv = threading.Condition()
        self._pending: list[tuple[Any, str, Any, Future]] = []
        self._active = 0
        self._stop = False
        self.batches: list[int] = []  # sizes of the device passes issued
        self._thread = threading.Thread(target=self._loop, name="batch-dispatch", daemon=True)
        self._thread.start()

    # -- clients ---------------------------------------------------------------
    def _submit(self, backend: Any, kind: str, request: Any):
        fut: Future = Future()
        with self._cv:
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

    def close(self) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify_all()
        self._thread.join()

    # -- dispatcher ------------------------------------------------------------
    def _loop(self) -> None:
        while True:
            with self._cv:
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
            self._dispatch(batch)

    def _dispatch(self, batch) -> None:
        groups: dict[tuple, list] = {}
        for backend, kind, req, fut in batch:
            key = (id(backend), kind) + ((tuple(req.stop), req.max_tokens) if kind == "gen" else ())
            groups.setdefault(key, []).append((backend, kind, req, fut))
        for items in groups.values():
            backend, kind = items[0][0], items[0][1]
            cap = len(backend.pool.streams)  # one KV stream per request of a pass
            for i in range(0, len(items), cap):
                chunk = items[i:i + cap]
                reqs = [it[2] for it in chunk]
                try:
                    if len(reqs) == 1:
                        one = (backend.generate_step if kind == "gen" else backend.score_step)(reqs[0])
                        res: list = [one]
                    elif kind == "gen":
                        res = backend.generate_steps(reqs)
                    else:
                        res = backend.score_steps(reqs)
                except BaseException as exc:
                    res = [exc] * len(chunk)
                self.batches.append(len(chunk))
                for (_, _, _, fut), r in zip(chunk, res):
                    fut.set_result(r)
