"""Pin the host-side mirror of the reference API against the reference's own
known answers (copied as literal expectations from its tests, cited) and,
when the reference package is mounted, against the reference functions on
randomised inputs."""

import dataclasses
import random

import numpy as np
import pytest

from paper_2504_07891_b200 import contract, domain, driver, pricing
from paper_2504_07891_b200.domain import (
    AcceptanceThreshold,
    Decision,
    EngineConfig,
    UtilityScore,
    decide_acceptance,
)


# ---------------------------------------------------------------- judge rule
@pytest.mark.parametrize("score,thr,want", [(8, 7, "Accept"), (7, 7, "Accept"),
                                            (0, 0, "Accept"), (9, 10, "Reject")])
def test_decide_acceptance_known_answers(score, thr, want):
    # test_core.py:41-52
    assert decide_acceptance(UtilityScore(score), AcceptanceThreshold(thr)).value == want


def test_decide_acceptance_monotone():
    # test_core.py:54-64: accepting at t implies accepting at every t' < t
    rng = random.Random(0)
    for _ in range(2000):
        s, t = rng.randint(0, 9), rng.randint(0, 10)
        d = decide_acceptance(UtilityScore(s), AcceptanceThreshold(t))
        assert (d is Decision.ACCEPT) == (s >= t)


@pytest.mark.parametrize("bad", [-1, 10, True, 3.0])
def test_score_validation(bad):
    with pytest.raises((ValueError, TypeError)):
        UtilityScore(bad)


def test_threshold_validation():
    with pytest.raises(ValueError):
        AcceptanceThreshold(11)
    with pytest.raises(TypeError):
        AcceptanceThreshold(False)


# ------------------------------------------------------------ extract_score
def test_extract_score_known_answers():
    # test_backends.py:149-167
    assert contract.extract_score({"7": -0.2, "8": -1.9, "3": -4.0}, "ignored") == UtilityScore(7)
    assert contract.extract_score({" 9": -0.5, "ok": -0.1, "42": -0.2}, "") == UtilityScore(9)
    assert contract.extract_score(None, "  8 because it checks out") == UtilityScore(8)
    with pytest.raises(contract.ScoreParseFailure):
        contract.extract_score({"ok": -0.1}, "no numerals here")


def test_extract_score_tie_first_wins():
    assert contract.extract_score({"4": -1.0, "6": -1.0}, "") == UtilityScore(4)
    assert contract.extract_score({"6": -1.0, "4": -1.0}, "") == UtilityScore(6)


def test_extract_score_matches_reference_random(stepspec):
    from stepspec.backends import base as rbase

    rng = np.random.default_rng(11)
    toks = [str(d) for d in range(10)] + [" 5", "5 ", "ok", "42", "x9", "", " "]
    for _ in range(500):
        k = int(rng.integers(0, 8))
        table = {str(t): float(rng.normal(-2, 1)) for t in rng.choice(toks, size=k)}
        text = "".join(rng.choice(list("ab 7c0"), size=int(rng.integers(0, 6))))
        try:
            want = rbase.extract_score(table or None, text).value
        except rbase.ScoreParseFailure:
            want = None
        try:
            got = contract.extract_score(table or None, text).value
        except contract.ScoreParseFailure:
            got = None
        assert got == want


# -------------------------------------------------- prefix token accounting
class _Counter(contract.Backend):
    def generate_step(self, request):
        raise NotImplementedError

    def score_step(self, request):
        raise NotImplementedError


def test_count_new_prompt_tokens_known_answers():
    # test_backends.py:175-196
    b = _Counter()
    assert contract.count_new_prompt_tokens("a b c", "a b c", b) == 0
    prev = "problem statement so far"
    assert contract.count_new_prompt_tokens(prev, prev + " " + " ".join(f"w{i}" for i in range(70)), b) == 70
    assert contract.count_new_prompt_tokens("x y", "a b c", b) == 3
    rng = np.random.default_rng(5)
    text = " ".join(f"tok{i}" for i in range(200))
    for _ in range(200):
        cut = int(rng.integers(0, len(text)))
        assert contract.count_new_prompt_tokens(text[:cut], text, b) == len(text[cut:].split())


# ------------------------------------------------------------- segmentation
def test_segment_step_known_answers():
    # test_engine.py:35-55
    cfg = EngineConfig()
    seg = driver.segment_step("Compute 2+3 = 5.\n\nNext,", cfg)
    assert (seg.text, seg.end_think, seg.truncated) == ("Compute 2+3 = 5.\n\n", False, False)
    seg = driver.segment_step("one two three four five six", dataclasses.replace(cfg, max_step_tokens=4))
    assert (seg.text, seg.truncated) == ("one two three four", True)
    seg = driver.segment_step("last point.</think>\nanswer text", cfg)
    assert (seg.text, seg.end_think) == ("last point.", True)
    seg = driver.segment_step("a.\nb</think>", cfg)
    assert (seg.text, seg.end_think) == ("a.\n", False)


def test_segment_step_matches_reference_random(stepspec):
    from stepspec import engine as reng
    from stepspec.core import EngineConfig as RConfig

    rng = random.Random(3)
    alphabet = ["a", "b", " ", "\n", ".", "!", "?", "</think>", "w1", "\n\n"]
    for _ in range(2000):
        text = "".join(rng.choice(alphabet) for _ in range(rng.randint(0, 30)))
        mst = rng.randint(1, 8)
        mine = driver.segment_step(text, EngineConfig(max_step_tokens=mst))
        ref = reng.segment_step(text, RConfig(max_step_tokens=mst))
        assert (mine.text, mine.end_think, mine.truncated) == (ref.text, ref.end_think, ref.truncated)


def test_force_first_n():
    # test_engine.py:70-78
    assert not any(driver.force_first_n(EngineConfig(), i) for i in range(50))
    cfg = EngineConfig(force_first_n=10)
    assert driver.force_first_n(cfg, 9) and not driver.force_first_n(cfg, 10)


# --------------------------------------------------------- prompts / tokens
def test_prompt_layout_matches_reference(stepspec):
    from stepspec import prompts as rp

    assert domain.VERIFY_PROMPT_V1 == rp.VERIFY_PROMPT_V1
    assert domain.verification_sections() == rp.verification_sections()
    assert (domain.VERIFY_HEAD_TOKENS, domain.VERIFY_TAIL_TOKENS) == (rp.VERIFY_HEAD_TOKENS,
                                                                      rp.VERIFY_TAIL_TOKENS)
    for cot in ("", "a b.\n", "x</think>y"):
        for done in (False, True):
            p = domain.render_generation_prompt("prob lem", cot, done)
            assert p == rp.render_generation_prompt("prob lem", cot, done)
            assert domain.split_generation_prompt(p) == rp.split_generation_prompt(p)
    rng = random.Random(1)
    for _ in range(300):
        t = "".join(rng.choice("ab \n\t.") for _ in range(rng.randint(0, 40)))
        n = rng.randint(-1, 12)
        assert domain.truncate_tokens(t, n) == rp.truncate_tokens(t, n)
        assert domain.count_tokens(t) == rp.count_tokens(t)


def test_verify_overhead_constants():
    # prompts.py:98 measured 14 / 38
    assert (domain.VERIFY_HEAD_TOKENS, domain.VERIFY_TAIL_TOKENS) == (14, 38)


# ---------------------------------------------------------- value round trips
def test_json_round_trips_match_reference(stepspec):
    from stepspec import core as rc

    cfg = EngineConfig(threshold=AcceptanceThreshold(3), seed=9, max_step_tokens=17)
    assert cfg.to_dict() == rc.EngineConfig.from_dict(cfg.to_dict()).to_dict()
    assert EngineConfig.from_dict(cfg.to_dict()) == cfg
    step = domain.ReasoningStep(2, "x y", 2, domain.StepProducer.SPECULATOR, UtilityScore(5), True,
                                domain.LatencyBreakdown(0.1, 0.2, 0.0))
    assert rc.ReasoningStep.from_dict(step.to_dict()).to_dict() == step.to_dict()
    assert domain.ReasoningStep.from_dict(step.to_dict()) == step
    st = domain.TrajectoryState("p", [step], 2, domain.Phase.DONE, 10, "ans")
    assert rc.TrajectoryState.from_dict(st.to_dict()).to_dict() == st.to_dict()
    m = domain.RunMetrics(1.5, 3, 0.5, 1, False, domain.Scheme.SPEC_REASON, True)
    assert rc.RunMetrics.from_dict(m.to_dict()).to_dict() == m.to_dict()
    prof = domain.BackendProfile("n", domain.BackendRole.BASE, 0.01, 100.0)
    assert rc.BackendProfile.from_dict(prof.to_dict()).to_dict() == prof.to_dict()


def test_metrics_validation():
    with pytest.raises(ValueError):
        domain.RunMetrics(1.0, 1, 0.5, 0, False, domain.Scheme.BASE_ONLY, False)
    with pytest.raises(ValueError):
        domain.RunMetrics(1.0, 1, 1.5, 0, False, domain.Scheme.SPEC_REASON, False)


# ------------------------------------------------------------------- seeds
def test_seed_derivation_matches_reference(stepspec):
    from stepspec import bench as rb
    from stepspec import seeding as rs
    from stepspec import specdecode as rsd

    for parts in [("a", 1), ("trajectory", 0, "task0001", 3), (b"x", None, 2.5)]:
        assert pricing.derive_seed(*parts) == rs.derive_seed(*parts)
        assert pricing.derive_rng(*parts).random() == rs.derive_rng(*parts).random()
    assert pricing.trajectory_seed(7, "task0003", 2) == rb.trajectory_seed(7, "task0003", 2)
    for n, g, a in [(0, 5, 0.8), (13, 5, 0.8), (40, 3, 0.0), (25, 7, 1.0)]:
        assert pricing.simulate_regen_rounds(n, g, a, pricing.derive_rng("r", n)) == \
            rsd.simulate_regen_rounds(n, g, a, rs.derive_rng("r", n))
