"""The driver (``driver.py``) against the reference engine (``engine.py``).

1. Both engines drive the reference's own simulated backends (its test
   fixtures, ``tests/conftest.py:17-29``) over a grid of knobs; every state,
   trace record, metric and latency float must be identical.
2. The reference engine drives the CPU oracle backend bound to the
   reference's types, and our driver drives the same oracle with our types:
   identical trajectories.  This is how the committed golden fixtures were
   produced (tests/golden/make_golden.py).
3. Engine-level invariants from the reference's test suite (forced reject ==
   pure base, threshold 0 == all speculator, parse failure == reject, error
   context) hold for our driver.
"""

import dataclasses
import itertools

import pytest

from paper_2504_07891_b200 import contract, driver
from paper_2504_07891_b200.domain import (AcceptanceThreshold, BackendProfile, BackendRole,
                                          EngineConfig, StepProducer, UtilityScore)


def _as_plain(result):
    return {
        "state": result.state.to_dict(),
        "trace": result.trace,
        "metrics": result.metrics.to_dict(),
        "rejected": [s.to_dict() for s in result.rejected_steps],
        "answer_latency_s": result.answer_latency_s,
        "actions": [o.action.value for o in result.outcomes],
    }


@pytest.fixture(scope="module")
def sim(stepspec):
    from stepspec.backends.simulated import SimulatedBackend
    from stepspec.simlab import DEFAULT_BASE_SPEC, DEFAULT_JUDGE_SPEC, DEFAULT_SMALL_SPEC, make_tasks

    small = SimulatedBackend(DEFAULT_SMALL_SPEC, seed=0)
    base = SimulatedBackend(DEFAULT_BASE_SPEC, judge_spec=DEFAULT_JUDGE_SPEC, seed=0)
    return small, base, make_tasks(20, 12, seed=7)


GRID = list(itertools.product((0, 3, 7, 10), (0, 3), (False, True), (8192, 40)))


@pytest.mark.parametrize("thr,force,hier,budget", GRID)
def test_driver_equals_reference_engine_on_simulator(stepspec, sim, thr, force, hier, budget):
    from stepspec import engine as reng
    from stepspec.core import AcceptanceThreshold as RThr
    from stepspec.core import EngineConfig as RConfig

    small, base, tasks = sim
    for i, task in enumerate(tasks[:4]):
        kw = dict(force_first_n=force, hierarchical=hier, token_budget=budget, seed=31 * i + thr)
        ref = reng.run_trajectory(RConfig(threshold=RThr(thr), **kw), task.problem_text(), small, base)
        mine = driver.run_trajectory(EngineConfig(threshold=AcceptanceThreshold(thr), **kw),
                                     task.problem_text(), small, base)
        assert _as_plain(mine) == _as_plain(ref)


@pytest.mark.parametrize("which,spec", [("base", False), ("small", False), ("base", True)])
def test_vanilla_equals_reference_on_simulator(stepspec, sim, which, spec):
    from stepspec import engine as reng
    from stepspec.core import EngineConfig as RConfig

    small, base, tasks = sim
    backend = base if which == "base" else small
    for i, task in enumerate(tasks[:5]):
        kw = dict(seed=100 + i, token_budget=60 if i % 2 else 8192)
        ref = reng.run_vanilla(RConfig(**kw), task.problem_text(), backend,
                               draft=small if spec else None, token_speculative=spec)
        mine = driver.run_vanilla(EngineConfig(**kw), task.problem_text(), backend,
                                  draft=small if spec else None, token_speculative=spec)
        assert _as_plain(mine) == _as_plain(ref)


def test_validate_trajectory_accepts_reference_runs(stepspec, sim):
    small, base, tasks = sim
    cfg = EngineConfig(seed=3)
    res = driver.run_trajectory(cfg, tasks[0].problem_text(), small, base)
    driver.validate_trajectory(res, cfg)
    bad = dataclasses.replace(res, answer_latency_s=res.answer_latency_s + 1.0)
    with pytest.raises(ValueError):
        driver.validate_trajectory(bad, cfg)


# -------------------------------------------------------- oracle backends
def test_reference_engine_drives_oracle_backend_identically(stepspec):
    """Drop-in: the reference's run_trajectory accepts our backend (bound to
    its types) and yields the same trajectory as our driver."""
    from oracle.ref_engine import oracle_backend
    from paper_2504_07891_b200.host import reference_types
    from paper_2504_07891_b200.vocab import shared_vocab
    from stepspec import engine as reng
    from stepspec.core import AcceptanceThreshold as RThr
    from stepspec.core import EngineConfig as RConfig

    T = reference_types(stepspec)
    r_small = oracle_backend("tiny-draft", BackendRole.SMALL, types=T)
    r_base = oracle_backend("tiny-base", BackendRole.BASE, types=T)
    m_small = oracle_backend("tiny-draft", BackendRole.SMALL)
    m_base = oracle_backend("tiny-base", BackendRole.BASE)
    v = shared_vocab(4096)
    kw = dict(temperature=0.0, max_step_tokens=32, token_budget=128)
    for p in range(2):
        prob = v.problem(64, p)
        ref = reng.run_trajectory(RConfig(threshold=RThr(7), **kw), prob, r_small, r_base)
        mine = driver.run_trajectory(EngineConfig(threshold=AcceptanceThreshold(7), **kw), prob,
                                     m_small, m_base)
        assert driver.trace_signature(mine) == driver.trace_signature(ref)
        reng.validate_trajectory(ref, RConfig(threshold=RThr(7), **kw))


# -------------------------------------------------- engine-level invariants
class _Scripted(contract.Backend):
    """Deterministic fake: fixed step text; scores from a list (None = parse failure)."""

    def __init__(self, role, scores=(), fail_after=None):
        self.profile = BackendProfile(f"fake-{role.value}", role, 0.01, 1000.0)
        self.scores = list(scores)
        self.calls = 0
        self.fail_after = fail_after

    def generate_step(self, request):
        self.calls += 1
        if self.fail_after is not None and self.calls > self.fail_after:
            raise contract.TransportError("boom")
        word = "s" if self.profile.role == BackendRole.SMALL else "b"
        answering = request.prompt.endswith("</think>\n")
        text = "answer 42" if answering else f"{word}{self.calls} x y.\n"
        return contract.GenerationResult(text, len(text.split()), contract.FinishReason.STOP,
                                          measured_latency_s=0.001)

    def score_step(self, request):
        s = self.scores.pop(0) if self.scores else 9
        if s is None:
            raise contract.ScoreParseFailure("no digit")
        return UtilityScore(s)


def test_parse_failure_is_reject():
    # test_engine.py:223-249
    small, base = _Scripted(BackendRole.SMALL), _Scripted(BackendRole.BASE, scores=[None, None, 9])
    res = driver.run_trajectory(EngineConfig(token_budget=12), "prob", small, base)
    assert [s.producer for s in res.state.retained_steps][:2] == [StepProducer.BASE] * 2
    assert res.rejected_steps[0].score is None
    driver.validate_trajectory(res, EngineConfig(token_budget=12))


def test_threshold_extremes():
    cfg10 = EngineConfig(threshold=AcceptanceThreshold(10), token_budget=16)
    res = driver.run_trajectory(cfg10, "p", _Scripted(BackendRole.SMALL), _Scripted(BackendRole.BASE))
    assert all(s.producer == StepProducer.BASE for s in res.state.retained_steps)
    cfg0 = EngineConfig(threshold=AcceptanceThreshold(0), token_budget=16)
    res = driver.run_trajectory(cfg0, "p", _Scripted(BackendRole.SMALL), _Scripted(BackendRole.BASE))
    assert all(s.producer == StepProducer.SPECULATOR for s in res.state.retained_steps)
    assert res.rejected_steps == []


def test_error_context_and_roles():
    # test_engine.py:252-292
    with pytest.raises(ValueError):
        driver.run_trajectory(EngineConfig(), "p", _Scripted(BackendRole.BASE), _Scripted(BackendRole.BASE))
    small = _Scripted(BackendRole.SMALL, fail_after=2)
    with pytest.raises(contract.TransportError, match="step 2 of problem"):
        driver.run_trajectory(EngineConfig(threshold=AcceptanceThreshold(0)), "p\nmore", small,
                              _Scripted(BackendRole.BASE))


def test_session_steps_equal_run_trajectory(stepspec, sim):
    small, base, tasks = sim
    cfg = EngineConfig(seed=4, token_budget=120)
    whole = driver.run_trajectory(cfg, tasks[1].problem_text(), small, base)
    sess = driver.SpecReasonSession(cfg, tasks[1].problem_text(), small, base)
    n = 0
    while sess.step() is not None:
        n += 1
    res = sess.finish()
    assert n == len(res.outcomes)
    assert _as_plain(res) == _as_plain(whole)
