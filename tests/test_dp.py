"""Request-level data parallelism (config C5, ``paper_2504_07891_b200/dp.py``):
problems are split by ``problem_id`` and seeded by ``trajectory_seed``
(``bench.py:216-218``), so every problem's trajectory is identical whether
one rank or two ranks (gloo, CPU oracle backends) run the sweep; the sweep's
forced-reject cell equals BaseOnly (``test_acceptance.py:104-113``)."""

import os
import pickle
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig, Scheme
from paper_2504_07891_b200.dp import (cells, check_forced_reject, gather, partition,
                                      problem_ids, run_partition)

N_PROBLEMS = 4
THRESHOLDS = (3, 7, 10)
CFG = dict(temperature=0.0, max_step_tokens=32, token_budget=96)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _backends():
    from oracle.ref_engine import oracle_backend
    from paper_2504_07891_b200.domain import BackendRole

    return (oracle_backend("tiny-draft", BackendRole.SMALL),
            oracle_backend("tiny-base", BackendRole.BASE))


def _run(rank: int, world: int):
    # one thread everywhere: the oracle's fp32 sums then run in one order on
    # every rank (a different BLAS split could flip a bf16 rounding)
    torch.set_num_threads(1)
    small, base = _backends()
    ids = partition(problem_ids(N_PROBLEMS), rank, world)
    cfg = EngineConfig(threshold=AcceptanceThreshold(7), **CFG)
    return run_partition(ids, small, base, cfg, THRESHOLDS,
                         schemes=(Scheme.SPEC_REASON, Scheme.BASE_ONLY))


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = gather(_run(rank, world), dist)
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(recs, f)
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_ids_once():
    ids = problem_ids(64)
    for world in (1, 2, 3, 8):
        parts = [partition(ids, r, world) for r in range(world)]
        assert sum(parts, []) == ids
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_world2_records_equal_world1(tmp_path):
    threads = torch.get_num_threads()
    try:
        one = gather(_run(0, 1))
    finally:
        torch.set_num_threads(threads)
    out = tmp_path / "dp2.pkl"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    with open(out, "rb") as f:
        two = pickle.load(f)
    assert [r.key() for r in one] == [r.key() for r in two]
    assert [r.outcome() for r in one] == [r.outcome() for r in two]
    assert len(one) == N_PROBLEMS * (len(THRESHOLDS) + 1)
    assert check_forced_reject(one) == N_PROBLEMS
    c = cells(one)
    assert c["SpecReason@10"]["accepted_fraction"] == 0.0
    assert c["BaseOnly@-1"]["n"] == N_PROBLEMS
