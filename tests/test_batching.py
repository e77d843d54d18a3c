"""Concurrent trajectories through ``BatchScheduler``: every
trajectory equals the one it produces alone, and the device calls were
actually batched.  CPU oracle backends."""

from oracle.ref_engine import oracle_backend
from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
from paper_2504_07891_b200.batching import BatchScheduler
from paper_2504_07891_b200.domain import BackendRole
from paper_2504_07891_b200.driver import run_trajectory
from paper_2504_07891_b200.vocab import shared_vocab


def _pair(n_streams):
    return (oracle_backend("tiny-draft", BackendRole.SMALL, n_streams=n_streams),
            oracle_backend("tiny-base", BackendRole.BASE, n_streams=n_streams))


def test_concurrent_trajectories_equal_serial():
    cfg = EngineConfig(threshold=AcceptanceThreshold(5), temperature=0.0, token_budget=96,
                       max_step_tokens=16)
    small, base = _pair(8)
    v = shared_vocab(small.engine.spec.vocab_text)
    problems = [v.problem(32, 100 + k) for k in range(3)]
    sched = BatchScheduler(small, base)
    try:
        got = sched.run([lambda s, b, p=p: run_trajectory(cfg, p, s, b) for p in problems])
    finally:
        sched.close()
    s2, b2 = _pair(8)
    for p, g in zip(problems, got):
        assert not isinstance(g, BaseException), g
        want = run_trajectory(cfg, p, s2, b2)
        key = lambda r: [(o.step.text, o.step.producer, o.step.score, o.step.accepted)  # noqa: E731
                         for o in r.outcomes]
        assert key(g) == key(want)
        assert g.metrics.thinking_tokens == want.metrics.thinking_tokens
    assert max(sched.batches) > 1  # requests of different trajectories shared passes
