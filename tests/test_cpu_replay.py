"""The CPU cost replay behind ``bench.py``'s ``cpu_baseline`` and the
reference arm (``oracle/cpu_replay.py``): a bounded per-call sample (a
fraction of the layers, at most ``decode_cap`` decode steps, scaled back)
must estimate the full-depth, every-token cost of the same call."""

import pytest

from oracle.cpu_replay import CpuReplay
from paper_2504_07891_b200.shapes import get_spec


@pytest.mark.slow
def test_sampled_cost_tracks_full_cost():
    spec = {"r1-1.5b": get_spec("r1-1.5b")}
    full = CpuReplay(spec, 3072)
    samp = CpuReplay(spec, 3072, layer_frac=1 / 7, decode_cap=4)
    full.warm()
    samp.warm()
    calls = [{"model": "r1-1.5b", "kind": "gen", "start": 2000, "fresh": 40, "n_gen": 24},
             {"model": "r1-1.5b", "kind": "score", "start": 2000, "fresh": 96, "n_gen": 1}]
    for c in calls:
        f = min(full.run(c) for _ in range(2))
        s = min(samp.run(c) for _ in range(2))
        assert 0.65 < s / f < 1.5, (c["kind"], f, s)
    assert samp.wall_s < full.wall_s / 2  # the sample is cheaper than what it prices
    assert "4 of 28 layers" in samp.sample_text()
