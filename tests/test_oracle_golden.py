"""The CPU oracle + our driver reproduce the golden trajectories that the
unmodified reference engine produced (tests/golden/make_golden.py), and the
golden set itself satisfies the reference's acceptance criteria C1/C2
(test_acceptance.py:104-126)."""

import json
from pathlib import Path

import pytest

from oracle.ref_engine import oracle_backend
from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig, run_trajectory, run_vanilla
from paper_2504_07891_b200.domain import BackendRole
from paper_2504_07891_b200.driver import trace_signature, validate_trajectory
from paper_2504_07891_b200.vocab import shared_vocab

GOLDEN = json.loads((Path(__file__).parent / "golden" / "c1_trajectories.json").read_text())


def _norm(sig):
    return json.loads(json.dumps(sig))


def _cases(kind):
    return [c for c in GOLDEN["cases"] if c["kind"] == kind]


@pytest.mark.parametrize("case", _cases("spec_reason")[:3] + _cases("spec_reason")[6:8],
                         ids=lambda c: f"thr{c['threshold']}-p{c['problem_seed']}")
def test_driver_with_oracle_reproduces_golden(case):
    v = shared_vocab(4096)
    small = oracle_backend("tiny-draft", BackendRole.SMALL)
    base = oracle_backend("tiny-base", BackendRole.BASE, threshold=case["threshold"])
    cfg = EngineConfig(threshold=AcceptanceThreshold(case["threshold"]), **GOLDEN["config"])
    res = run_trajectory(cfg, v.problem(64, case["problem_seed"]), small, base)
    validate_trajectory(res, cfg)
    assert _norm(trace_signature(res)) == case["signature"]


def test_golden_forced_reject_equals_pure_base():
    spec = {c["problem_seed"]: c for c in _cases("spec_reason") if c["threshold"] == 10}
    for van in _cases("vanilla_base"):
        s = spec[van["problem_seed"]]["signature"]
        assert [st[1] for st in s["steps"]] == [st[1] for st in van["signature"]["steps"]]
        assert s["answer"] == van["signature"]["answer"]
        assert all(a == "RejectedThenRegenerated" for a in s["actions"])


def test_golden_threshold_zero_all_speculator():
    for c in _cases("spec_reason"):
        if c["threshold"] == 0:
            assert all(st[3] == "Speculator" for st in c["signature"]["steps"])
            assert c["signature"]["rejected"] == []


def test_golden_exercises_both_branches():
    sr = [c for c in _cases("spec_reason") if c["threshold"] == 7]
    acc = sum(1 for c in sr for st in c["signature"]["steps"] if st[3] == "Speculator")
    rej = sum(len(c["signature"]["rejected"]) for c in sr)
    assert acc > 5 and rej > 5


def test_vanilla_base_matches_golden():
    v = shared_vocab(4096)
    case = _cases("vanilla_base")[0]
    cfg = EngineConfig(threshold=AcceptanceThreshold(10), **GOLDEN["config"])
    res = run_vanilla(cfg, v.problem(64, case["problem_seed"]), oracle_backend("tiny-base", BackendRole.BASE))
    assert _norm(trace_signature(res)) == case["signature"]
