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


def test_reference_run_sweep_through_scheduler(stepspec, tmp_path):
    """The reference's own thread-pooled sweep driving the proxies."""
    from stepspec.bench import Knob, SweepSpec, run_sweep
    from stepspec.core import AcceptanceThreshold as RefThreshold
    from stepspec.core import EngineConfig as RefConfig
    from stepspec.core import Scheme
    from stepspec.simlab import make_tasks

    from paper_2504_07891_b200.host import reference_types

    T = reference_types(stepspec)
    small = oracle_backend("tiny-draft", BackendRole.SMALL, n_streams=8, types=T)
    base = oracle_backend("tiny-base", BackendRole.BASE, n_streams=8, types=T)
    sched = BatchScheduler(small, base).clients(3)
    try:
        cfg = RefConfig(threshold=RefThreshold(5), temperature=0.0, token_budget=48,
                        max_step_tokens=12)
        res = run_sweep(SweepSpec(knob=Knob.THRESHOLD, values=(5,), base_config=cfg, repeats=1),
                        make_tasks(3, 2, seed=0), sched.small, sched.base,
                        schemes=(Scheme.SPEC_REASON,), parallelism=3, output_dir=tmp_path)
    finally:
        sched.clients(-3)
        sched.close()
    assert len(res.records) == 3
    assert max(sched.batches) > 1


def test_open_generation_streams_are_not_reused():
    """A stream held by a continuously batched generation is never handed to
    another request, even when it is the least recently used one."""
    small = oracle_backend("tiny-draft", BackendRole.SMALL, n_streams=3)
    v = shared_vocab(small.engine.spec.vocab_text)
    from paper_2504_07891_b200.contract import GenerationRequest
    from paper_2504_07891_b200.domain import render_generation_prompt

    g = small.gen_open(GenerationRequest(prompt=render_generation_prompt(v.problem(16, 1), ""),
                                         max_tokens=4))
    held = g["stream"]
    for k in range(6):  # unrelated prompts cycle through the other streams
        st, _ = small.pool.acquire(v.encode(render_generation_prompt(v.problem(16, 50 + k), "")))
        assert st is not held
    small.gen_release(g)
    assert held not in small.pool.busy
