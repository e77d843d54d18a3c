"""SpecReason inner-loop benchmark (BASELINE.json metric: CoT tokens/s and ms
per reasoning step, draft + verify + fallback).

Workload (default, N=1): configuration C3 -- R1-Distill-1.5B-shape draft +
QwQ-32B-shape base, random-init bf16 (seeded, with the documented successor /
judge weight circuits of ``shapes.py``), greedy, threshold 7, 8192-token
thinking budget, 64-word synthetic problems (``dp.problem_text``).  One
*step* is one iteration of the SpecReason thinking loop driven through the
public API (``driver.SpecReasonSession`` over two ``B200Backend``s): the draft
decodes a step, the base scores it in one prefill pass, and on reject the base
regenerates it.  The K timed steps are split over P = 4 windows
(``--windows``), one per problem (task0000..), spread over the trajectory:
an untimed fast-forward runs window i's trajectory to 0.75 * budget * (i +
1/2) / P CoT tokens (768, 2304, 3840, 5376 of an 8 K budget: the acceptance
rate drifts down along a trajectory, so windows that all started at one
point over-weighted it), then (first window only) W warm-up steps, then the
window's share of the K timed steps.  The loop metric follows the
acceptance rate of the timed steps, so several problems' windows at several
depths give a steadier number than one.

Reported (one JSON line, rank 0):
  value      CoT tokens / s over the K timed steps, device time (sum of the
             CUDA-event durations of every native call: prefill + decode +
             readout), whole job = all ranks' tokens / max rank time
  e2e        the same metric end to end: wall time of the K steps through the
             public API (tokenisation, the Python driver, H2D of ids, D2H of
             results), CUDA events + synchronize around the region
  roofline   the kernel instance with the largest device time in the window
             (draft decode, base decode, or base prefill = verify + fallback
             prompts): algorithmic bytes / flops (shapes.py) over
             its CUDA-event time, against MEASURED_PEAKS.json; ``kernels``
             lists every instance
  cpu_baseline  the oracle's arithmetic for the first timed steps' recorded
             calls (full shapes, full depth, real context lengths) executed on
             the host cores (``oracle/cpu_replay.py``), >= ~20 s of CPU work
Multi-GPU (torchrun): ``--mode dp`` splits a fixed problem set by problem id
(``dp.partition``; no collective on the data path, scaling "weak");
``--mode tp`` shards the base over the ranks (C4).
``--impl reference`` runs the unmodified reference engine (``baseline/_ref``)
over the recorded trajectories of this benchmark's windows (``bench_data/``),
pricing every warm-up and timed step's calls on the host cores (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

METRIC = "CoT tokens/sec & ms per reasoning step (draft+verify+fallback) at 1–8 B200"
UNIT = "CoT tokens/s"
WORKLOADS = {
    "1.5b+7b": "C2: R1-Distill-1.5B-shape draft + Qwen2.5-7B-shape base, random-init bf16, 4K-token CoT, batch 1",
    "1.5b+32b": "C3: R1-1.5B-shape draft + QwQ-32B-shape base, random-init bf16, 8K-token CoT, threshold 7, batch 1",
    "tiny": "C1: tiny random-init pair (draft 2L d=128 + base 4L d=256), greedy, threshold 7",
}


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "src": "measured (MEASURED_PEAKS.json)"}
    # /opt/skills/guides/B200_PROFILING.md fallbacks
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1590.0,
            "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int) -> None:
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self) -> None:
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:  # noqa: BLE001 - clocks are best effort
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, v in zip(names, r[2:]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()  # more ranks than GPUs: share (testing)
    if world > 1:
        import torch.distributed as dist

        # the data path has no torch collective: DP ranks are independent and
        # TP uses the library's own NCCL communicator (only its 128-byte id
        # travels through torch.distributed), so gloo carries the few scalars
        dist.init_process_group("gloo", rank=rank, world_size=world)
        return dist, rank, world, local
    return None, 0, 1, local


def _reduce_max(dist, v: float) -> float:
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _reduce_sum(dist, v: float) -> float:
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class StepSource:
    """Endless sequence of SpecReason steps over back-to-back trajectories of
    the problems ``problem_ids`` (``dp.problem_text``)."""

    def __init__(self, small, base, config, problem_ids, vocab) -> None:
        from paper_2504_07891_b200.driver import SpecReasonSession

        self.cls = SpecReasonSession
        self.small, self.base, self.config = small, base, config
        self.problem_ids = list(problem_ids)
        self.vocab = vocab
        self.k = 0
        self.trajectories = 0
        self.session = None
        self.problems: list[str] = []
        self._new()

    def _new(self) -> None:
        from paper_2504_07891_b200.dp import problem_text

        pid = self.problem_ids[self.k % len(self.problem_ids)]
        self.k += 1
        text = problem_text(self.vocab, pid)
        self.problems.append(text)
        self.session = self.cls(self.config, text, self.small, self.base)
        self.trajectories += 1

    def step(self):
        while True:
            out = self.session.step()
            if out is not None:
                return out
            self._new()

    def fast_forward(self, cot_tokens: int) -> int:
        """Untimed steps until the current trajectory's CoT holds
        ``cot_tokens`` tokens (the timed window then sits mid-trajectory)."""
        n = 0
        while self.session.run.state.thinking_tokens_used < cot_tokens and self.session.thinking:
            if self.session.step() is None:
                break
            n += 1
        return n


# ------------------------------------------------------------- rooflines --
def kernel_lines(ds, db, names, peaks, sustained: bool) -> list[dict]:
    """Per kernel instance of the window: device ms, algorithmic work (SURVEY
    §8d), achieved rate and roofline fraction."""
    bw = peaks["hbm_gbs"]
    tf = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"]
    out = []
    for who, st, model in (("draft", ds, names[0]), ("base", db, names[1])):
        if st.decode_ms > 0:
            gbs = st.decode_bytes / (st.decode_ms * 1e-3) / 1e9
            out.append({"kernel": f"decode_mk_kernel ({who} {model} greedy decode, persistent)",
                        "instance": f"{who}_decode", "ms": round(st.decode_ms, 2),
                        "tokens": st.decode_tokens,
                        "bytes_per_token": round(st.decode_bytes / max(1, st.decode_tokens)),
                        "bound": "hbm", "achieved": round(gbs, 1), "peak": bw, "unit": "GB/s",
                        "frac": round(gbs / bw, 4)})
        if st.prefill_ms > 0:
            t = st.prefill_ms * 1e-3
            hbm_t = st.prefill_bytes / (bw * 1e9)
            ten_t = st.prefill_flops / (tf * 1e12)
            if ten_t > hbm_t:
                ach, peak, unit, bound = st.prefill_flops / t / 1e12, tf, "TFLOP/s", "tensor"
            else:
                ach, peak, unit, bound = st.prefill_bytes / t / 1e9, bw, "GB/s", "hbm"
            out.append({"kernel": f"prefill pass ({who} {model}: gemm_tc_persistent + "
                                  "attn_prefill_umma + epilogues"
                                  + (" + readout" if who == "base" else "") + ")",
                        "instance": f"{who}_prefill", "ms": round(st.prefill_ms, 2),
                        "rows": st.prefill_tokens, "bytes": round(st.prefill_bytes),
                        "flops": round(st.prefill_flops), "bound": bound,
                        "achieved": round(ach, 1), "peak": peak, "unit": unit,
                        "frac": round(ach / peak, 4),
                        "tflops": round(st.prefill_flops / t / 1e12, 1)})
    return out


def _traffic(instance: str, model: str):
    """DRAM bytes per unit from the committed ncu --set full capture of that
    kernel instance (profiles/r02_ncu_traffic.json), else None."""
    p = ROOT / "profiles" / "r02_ncu_traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text()).get(f"{instance}:{model}")
    if not d:
        return None, None
    return d["dram_bytes_per_unit"], d["source"]


# ------------------------------------------------------------- call trace --
def call_descriptors(backend, calls, model_key: str) -> list[dict]:
    """Compact, replayable form of recorded calls: what the engine received
    (text / count / finish or score) and what the device computed (context
    start, fresh rows, generated tokens)."""
    from paper_2504_07891_b200.host import FINISH_END_THINK, FINISH_STOP

    out = []
    for c in calls:
        start = len(c["prompt_ids"]) - c["fresh"]
        d = {"model": model_key, "kind": c["kind"], "prompt_len": len(c["prompt_ids"]),
             "start": start, "fresh": c["fresh"]}
        if c["kind"] == "gen":
            g = c["gen_ids"]
            fin = {FINISH_END_THINK: "EndThink", FINISH_STOP: "Stop"}.get(c["finish"], "Length")
            text_ids = g[:-1] if fin == "EndThink" else g
            d.update(n_gen=len(g), text=backend.vocab.render(text_ids), token_count=len(text_ids),
                     finish=fin)
        else:
            d.update(score=c["score"], n_gen=1)
            if c.get("catchup"):  # generation-stream rows prefilled in the same pass
                d.update(catchup=c["catchup"], catchup_start=c["catchup_start"])
        out.append(d)
    return out


def run_ours(args) -> None:
    from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.dp import partition, problem_ids
    from paper_2504_07891_b200.shapes import PAIRS, get_spec
    from paper_2504_07891_b200.vocab import shared_vocab

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    base_tp = None
    if args.mode == "tp":  # config C4: base sharded over the ranks, one shared trajectory
        from paper_2504_07891_b200.backend import TensorParallel

        base_tp = TensorParallel.from_dist() if dist is not None else TensorParallel.single()
    extra = {"n_streams": 2 * args.batch + 2, "max_tokens": 1024} if args.batch > 1 else {}
    record = rank == 0 and args.batch == 1
    small, base = build_pair(args.pair, seed=args.seed, max_ctx=args.budget + 512,
                             threshold=args.threshold, base_tp=base_tp, record=record, **extra)
    base.verify_template = args.verify_template
    if args.spec_gamma > 0:  # SpecReason+Decode: the draft proposes tokens inside base fallback
        base.attach_speculator(small, gamma=args.spec_gamma)
    names = PAIRS[args.pair]
    vocab = shared_vocab(get_spec(names[0]).vocab_text)
    cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                       token_budget=args.budget, max_step_tokens=args.max_step_tokens)
    # DP: this rank's block of a fixed problem set (problem-id partition, C5);
    # TP: every rank drives the same trajectories
    ids = problem_ids(args.problems)
    mine = ids if args.mode == "tp" else partition(ids, rank, world)
    ff = args.budget // 4 if args.ff_tokens < 0 else args.ff_tokens
    sched = None
    ff_steps = 0
    if args.batch > 1:  # B trajectories, each on its own thread, batched device passes
        from paper_2504_07891_b200.batching import BatchScheduler

        sched = BatchScheduler(small, base)
        srcs = [StepSource(sched.small, sched.base, cfg, mine[k::args.batch] or mine, vocab)
                for k in range(args.batch)]
        per = -(-args.steps // args.batch)

        def run_steps(n):
            res = sched.run([lambda s_, b_, src=src: [src.step() for _ in range(n)] for src in srcs])
            bad = [r for r in res if isinstance(r, BaseException)]
            if bad:
                raise bad[0]
            return [o for r in res for o in r]

        class _Multi:  # StepSource-like view for the shared reporting below
            trajectories = property(lambda self: sum(x.trajectories for x in srcs))

        src = _Multi()
        if ff > 0:
            sched.run([lambda s_, b_, src=src: src.fast_forward(ff) for src in srcs])
        run_steps(max(1, -(-args.warmup // args.batch)))

    stream = torch.cuda.current_stream()
    outcomes: list = []
    wins: list[dict] = []
    with ClockSampler(local) as clocks:
        if sched is not None:
            s0 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            outcomes = run_steps(per)
            e1.record(stream)
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            wall_ms = e0.elapsed_time(e1)
            ds = small.engine.stats.minus(s0[0])
            db = base.engine.stats.minus(s0[1])
        else:
            # the K timed steps are split over P windows, one per problem of
            # this rank's block, each after its own untimed fast-forward (the
            # W warm-up steps run before the first): the loop metric follows
            # the acceptance rate of the window, so several trajectories'
            # windows give a steadier number than one
            from paper_2504_07891_b200.backend import EngineStats

            P = max(1, min(args.windows, args.steps))
            per_w = [args.steps // P + (1 if i < args.steps % P else 0) for i in range(P)]
            wall_ms = 0.0
            ds, db = EngineStats(), EngineStats()
            for i, n in enumerate(per_w):
                wsrc = StepSource(small, base, cfg, [mine[i % len(mine)]], vocab)
                start = (len(small.calls), len(base.calls))
                ff_i = wsrc.fast_forward(window_ff(args, i, P))
                c_ff = (len(small.calls), len(base.calls))
                warm = []
                for _ in range(args.warmup if i == 0 else 0):
                    wsrc.step()
                    warm.append((len(small.calls), len(base.calls)))
                s0 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
                c0 = (len(small.calls), len(base.calls))
                if dist is not None:
                    dist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                outs, bounds = [], []
                e0.record(stream)
                for _ in range(n):
                    outs.append(wsrc.step())
                    bounds.append((len(small.calls), len(base.calls)))
                e1.record(stream)
                torch.cuda.synchronize()
                if dist is not None:
                    dist.barrier()
                wall_ms += e0.elapsed_time(e1)
                ds = ds.plus(small.engine.stats.minus(s0[0]))
                db = db.plus(base.engine.stats.minus(s0[1]))
                outcomes += outs
                ff_steps += ff_i
                wins.append({"src": wsrc, "start": start, "ff_steps": ff_i, "c_ff": c_ff,
                             "warm": warm, "c0": c0, "bounds": bounds, "outcomes": outs})

            class _Wins:  # StepSource-like view for the shared reporting below
                trajectories = sum(w["src"].trajectories for w in wins)

            src = _Wins()
    n_steps = len(outcomes)  # --batch B runs ceil(steps / B) steps on each trajectory

    tokens = sum(o.step.token_count for o in outcomes)
    dev_ms = ds.prefill_ms + ds.decode_ms + db.prefill_ms + db.decode_ms
    lat = [o.step.latency for o in outcomes]
    n_spec = sum(1 for o in outcomes if o.action.value == "AcceptedSpeculation")

    tot_tokens = _reduce_sum(dist, tokens) if args.mode == "dp" else tokens
    max_dev_ms = _reduce_max(dist, dev_ms)
    max_wall_ms = _reduce_max(dist, wall_ms)
    peaks = _peaks()
    kernels = kernel_lines(ds, db, names, peaks, sustained=True)
    dom = max(kernels, key=lambda k: k["ms"])
    traffic, traffic_src = _traffic(dom["instance"], names[0 if dom["instance"].startswith("draft") else 1])

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    ctx = [o.step.index for o in outcomes]
    result = {
        "metric": METRIC,
        "value": round(tot_tokens / (max_dev_ms * 1e-3), 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": n_steps,
        "warmup": args.warmup,
        "ms_per_step": round(max_wall_ms / n_steps, 3),
        "higher_is_better": True,
        "scaling": "weak" if args.mode == "dp" else "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded random-init weights with the shapes.py successor/judge circuits, "
                "seeded 64-word problems)",
        "config": bench_config(args, world),
        "e2e": {"value": round(tot_tokens / (max_wall_ms * 1e-3), 2), "unit": UNIT,
                "ms_per_step": round(max_wall_ms / n_steps, 3),
                "h2d_bytes_per_step": round((ds.h2d_bytes + db.h2d_bytes) / n_steps),
                "d2h_bytes_per_step": round((ds.d2h_bytes + db.d2h_bytes) / n_steps)},
        "breakdown_ms_per_step": {
            "speculate": round(1e3 * sum(x.speculate_s for x in lat) / n_steps, 3),
            "verify": round(1e3 * sum(x.verify_s for x in lat) / n_steps, 3),
            "fallback": round(1e3 * sum(x.fallback_s for x in lat) / n_steps, 3),
            "device": round(dev_ms / n_steps, 3)},
        "loop": {"tokens": tokens, "accepted_fraction": round(n_spec / len(outcomes), 3),
                 "trajectories": src.trajectories, "fast_forward_steps": ff_steps,
                 "first_step_index": min(ctx), "draft_decode_tokens": ds.decode_tokens,
                 "draft_decode_ms_per_token": round(ds.decode_ms / max(1, ds.decode_tokens), 4),
                 "base_decode_tokens": db.decode_tokens,
                 "base_decode_ms_per_token": round(db.decode_ms / max(1, db.decode_tokens), 4),
                 "base_prefill_rows": db.prefill_tokens, "base_prefill_ms": round(db.prefill_ms, 2)},
        "roofline": {**{k: dom[k] for k in ("kernel", "bound", "achieved", "peak", "unit", "frac")},
                     "instance": dom["instance"], "share_of_device_time": round(dom["ms"] / dev_ms, 4),
                     "peak_source": peaks["src"] + (", sustained bf16" if dom["unit"] == "TFLOP/s" else ""),
                     "algorithmic": "SURVEY §8d per-unit bytes/flops (shapes.ModelSpec.decode_bytes / "
                                    "prefill_cost) x units in the window / CUDA-event time of that "
                                    "kernel instance on its launch stream (sr_last_timing)",
                     "traffic": traffic, "traffic_source": traffic_src},
        "kernels": kernels,
        "gpu_launches": ds.launches + db.launches,
        **({"batching": {"trajectories_in_flight": args.batch,
                         "device_passes": len(sched.batches),
                         "mean_requests_per_pass": round(sum(sched.batches) / max(1, len(sched.batches)), 2)}}
           if sched is not None else {}),
        "clocks": clocks.summary(),
    }
    if record and args.dump_trace and wins:
        try:
            dump_trace(args, wins, small, base, names)
        except RuntimeError as exc:  # the line still prints; the trace is optional
            print(f"bench: no trace written: {exc}", file=sys.stderr, flush=True)
    if world == 1 and not args.no_cpu_baseline and record and wins:
        w0 = wins[0]
        result["cpu_baseline"] = cpu_baseline(args, small, base, names, w0["c0"], w0["bounds"],
                                              w0["outcomes"])
    print(json.dumps(result), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_sweep(args) -> None:
    """Config C5 as the reference's ``run_sweep`` (``bench.py:221-300``): the
    fixed problem set split by problem id over the ranks (``dp.partition``),
    every (threshold, problem) SpecReason trajectory plus BaseOnly, records
    gathered on rank 0; asserts threshold 10 == BaseOnly per problem
    (``test_acceptance.py:104-113``) and prints the per-cell summary."""
    from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig, Scheme
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.dp import (cells, check_forced_reject, gather, partition,
                                          problem_ids, run_partition)

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    small, base = build_pair(args.pair, seed=args.seed, max_ctx=args.budget + 512,
                             threshold=args.threshold)
    cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                       token_budget=args.budget, max_step_tokens=args.max_step_tokens)
    values = [int(x) for x in args.sweep.split(",")]
    mine = partition(problem_ids(args.problems), rank, world)
    t0 = time.perf_counter()
    recs = run_partition(mine, small, base, cfg, values, schemes=(Scheme.SPEC_REASON, Scheme.BASE_ONLY))
    secs = _reduce_max(dist, time.perf_counter() - t0)
    allrecs = gather(recs, dist)
    if rank == 0:
        n_checked = check_forced_reject(allrecs) if 10 in values else 0
        print(json.dumps({"sweep": values, "pair": args.pair, "budget": args.budget,
                          "problems": args.problems, "n_gpus": world,
                          "forced_reject_equals_base_only": n_checked,
                          "cells": cells(allrecs), "wall_s": round(secs, 1)}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def window_ff(args, i: int, P: int) -> int:
    """CoT tokens window i of P fast-forwards to (batch 1): spread over the
    first three quarters of the budget, or ``--ff-tokens`` for every window."""
    if args.ff_tokens >= 0:
        return args.ff_tokens
    return int(0.75 * args.budget * (i + 0.5) / P)


def bench_config(args, world: int) -> dict:
    """The ``config`` object both arms print (same_config)."""
    return {"workload": WORKLOADS[args.pair].replace("batch 1", f"batch {args.batch}"),
            "pair": args.pair, "threshold": args.threshold, "verify_template": args.verify_template,
            "spec_gamma": args.spec_gamma, "token_budget": args.budget,
            "max_step_tokens": args.max_step_tokens, "batch": args.batch,
            "timed_window": (f"the timed steps split over {max(1, min(args.windows, args.steps))} "
                             f"windows on the first problems of the block, each after an untimed "
                             f"fast-forward to "
                             f"{[window_ff(args, i, max(1, min(args.windows, args.steps))) for i in range(max(1, min(args.windows, args.steps)))]} "
                             f"CoT tokens (warm-up steps before the first)"
                             if args.batch == 1 else
                             f"after an untimed fast-forward of every trajectory to "
                             f"{args.budget // 4 if args.ff_tokens < 0 else args.ff_tokens} CoT "
                             f"tokens, then the warm-up steps"),
            "problems": f"task0000..task{args.problems - 1:04d} (dp.problem_text), split by id",
            "parallelism": (f"dp{world} (problem-id partition, no data-path collective"
                            + (f", {args.batch} concurrent trajectories per GPU sharing batched "
                               "device passes)" if args.batch > 1 else ")")
                            if args.mode == "dp" else
                            f"tp{world} (base sharded, NCCL all-reduce; draft replicated)"),
            "l2": "weights (3.5 + 65.5 GB) exceed L2 (126 MB) on every step: no flush needed"}


def dump_trace(args, wins, small, base, names) -> None:
    """Write every timed window's trajectory (``--impl reference`` replays
    them through the reference engine): per window the problem, the calls of
    its trajectory from its first call to the end of the window (fast-forward,
    warm-up and timed steps), where the window starts and the (small, base)
    call counts at the end of every warm-up / timed step -- all relative to
    the window's first call."""
    out = []
    for w in wins:
        if w["src"].trajectories != 1:
            raise RuntimeError("a window ran past its trajectory: raise --budget or lower --steps")
        s0 = w["start"]
        ends = [(a - s0[0], b - s0[1]) for a, b in w["warm"] + w["bounds"]]
        end = w["bounds"][-1]
        out.append({"problem": w["src"].problems[0], "fast_forward_steps": w["ff_steps"],
                    "warmup": len(w["warm"]), "steps": len(w["bounds"]),
                    "window_start": [w["c_ff"][0] - s0[0], w["c_ff"][1] - s0[1]],
                    "step_ends": [list(e) for e in ends],
                    "small": call_descriptors(small, small.calls[s0[0]:end[0]], names[0]),
                    "base": call_descriptors(base, base.calls[s0[1]:end[1]], names[1])})
    path = Path(args.dump_trace)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps({
        "pair": args.pair, "budget": args.budget, "threshold": args.threshold,
        "max_step_tokens": args.max_step_tokens, "windows": out}) + "\n")


def cpu_baseline(args, small, base, names, c0, bounds, outcomes) -> dict:
    """The oracle's arithmetic for the first timed steps' recorded calls, on
    the host cores (``oracle/cpu_replay.py``): steps are replayed in order
    until >= ``--cpu-seconds`` of CPU work (at least one step)."""
    from oracle.cpu_replay import CpuReplay
    from paper_2504_07891_b200.shapes import get_spec

    rep = CpuReplay({n: get_spec(n) for n in names}, max_ctx=args.budget + 1024)
    rep.warm()
    prev = c0
    secs = toks = n = 0
    for (cs, cb), o in zip(bounds, outcomes):
        calls = (call_descriptors(small, small.calls[prev[0]:cs], names[0])
                 + call_descriptors(base, base.calls[prev[1]:cb], names[1]))
        secs += sum(rep.run(c) for c in calls)
        toks += o.step.token_count
        n += 1
        prev = (cs, cb)
        if secs >= args.cpu_seconds:
            break
    return {"value": round(toks / secs, 3), "unit": UNIT, "cores": rep.threads, "kind": "port",
            "sample": (f"the first {n} timed steps ({toks} CoT tokens): every backend call of those "
                       f"steps (draft decode, verify prefill + readout, fallback decode) executed "
                       f"at the full {names[0]} / {names[1]} shapes and depth at its recorded "
                       f"context on {rep.threads} host threads (torch bf16 matmul, fp32 accumulate; "
                       f"oracle/cpu_replay.py)"),
            "ms_per_step": round(1e3 * secs / n, 1), "cpu_seconds": round(secs, 1)}


# ---------------------------------------------------------- reference arm --
def _reference_package():
    for root in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (root / "stepspec" / "__init__.py").exists():
            if str(root) not in sys.path:
                sys.path.insert(0, str(root))
            import stepspec

            return stepspec, str(root)
    return None, None


def _replay_backend_cls(stepspec):
    """A reference ``Backend`` (``backends/base.py:77-100``) that answers the
    reference engine with a recorded trajectory's results and, inside the
    window, spends the host-CPU cost of each call (``oracle/cpu_replay``):
    the engine's own clocks then measure that cost (``engine.py:199-202``,
    ``engine.py:284-294``)."""
    from stepspec.backends.base import (Backend, FinishReason, GenerationResult,
                                        ScoreParseFailure)
    from stepspec.core import UtilityScore

    class ReplayBackend(Backend):
        simulated = False

        def __init__(self, profile, calls, lo, hi, rep):
            self.profile = profile
            self.calls, self.lo, self.hi, self.rep = calls, lo, hi, rep
            self.i = 0
            self.cpu_s = 0.0
            self.cost: dict[int, float] = {}  # call index -> CPU seconds (scaled back)

        def _next(self, prompt: str) -> dict | None:
            if self.i >= len(self.calls):
                return None
            c = self.calls[self.i]
            if len(prompt.split()) != c["prompt_len"]:
                raise AssertionError(f"{self.profile.name} call {self.i}: the engine's prompt has "
                                     f"{len(prompt.split())} tokens, the trace {c['prompt_len']}")
            self.i += 1
            return c

        def _cost(self, c) -> float:
            if self.lo <= self.i - 1 < self.hi:
                t = self.rep.run(c)
                self.cpu_s += t
                self.cost[self.i - 1] = t
                return t
            return 0.0

        def generate_step(self, request):
            c = self._next(request.prompt)
            if c is None:  # past the recorded window: end thinking / empty answer
                return GenerationResult(text="", token_count=0, finish_reason=FinishReason.END_THINK)
            assert c["kind"] == "gen", c
            t = self._cost(c)
            return GenerationResult(text=c["text"], token_count=c["token_count"],
                                    finish_reason=FinishReason(c["finish"]), measured_latency_s=t)

        def score_step(self, request):
            from stepspec.prompts import render_verification_prompt

            c = self._next(render_verification_prompt(request.problem, request.cot_prefix,
                                                      request.candidate_step))
            if c is None:
                raise ScoreParseFailure("past the recorded window")
            assert c["kind"] == "score", c
            self._cost(c)
            if c["score"] < 0:
                raise ScoreParseFailure("no digit in the top-10 or the sampled token")
            return UtilityScore(c["score"])

    return ReplayBackend


def run_reference(args) -> None:
    """Reference arm: the unmodified reference engine (``run_trajectory``,
    ``engine.py:297``) drives replay backends over each recorded window's
    trajectory of this benchmark; every warm-up and timed step's calls are executed on the
    host cores at full model shape, on a bounded per-call sample of layers and
    decode steps scaled back per call (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    trace_path = Path(args.trace) if args.trace else ROOT / "bench_data" / f"{args.pair}_trace.json"
    stepspec, ref_root = _reference_package()
    why = None
    if stepspec is None:
        why = "reference package not installed in baseline/_ref"
    elif not trace_path.exists():
        why = f"no recorded trajectory {trace_path.name} for pair {args.pair}"
    if why:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    tr = json.loads(trace_path.read_text())
    for k in ("pair", "budget", "threshold", "max_step_tokens"):
        if tr[k] != getattr(args, k):
            print(json.dumps({"impl": "reference",
                              "unavailable": f"trace {k}={tr[k]} differs from --{k} {getattr(args, k)}"}))
            return
    wins = tr["windows"]
    P = max(1, min(args.windows, args.steps))
    per_w = [args.steps // P + (1 if i < args.steps % P else 0) for i in range(P)]
    warm_w = [args.warmup if i == 0 else 0 for i in range(P)]
    if len(wins) < P or any(w["warmup"] + w["steps"] < a + n for w, a, n in zip(wins, warm_w, per_w)):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"trace holds {[w['warmup'] + w['steps'] for w in wins]} steps per window, "
                          f"the run needs {[a + n for a, n in zip(warm_w, per_w)]}"}))
        return
    from oracle.cpu_replay import CpuReplay
    from paper_2504_07891_b200.shapes import PAIRS, get_spec
    from stepspec import engine as reng
    from stepspec.core import AcceptanceThreshold, BackendProfile, BackendRole, EngineConfig

    names = PAIRS[args.pair]
    t_start = time.perf_counter()
    # bounded sample per call (a layer sample and <= 16 decode steps, scaled
    # back per call): the steps' full-depth CPU work is tens of minutes
    rep = CpuReplay({n: get_spec(n) for n in names}, max_ctx=args.budget + 1024,
                    layer_frac=args.ref_layer_frac, decode_cap=args.ref_decode_cap)
    rep.warm()
    Replay = _replay_backend_cls(stepspec)
    prof = lambda n, r: BackendProfile(name=f"cpu-{n}", role=r, decode_s_per_token=1.0,  # noqa: E731
                                       prefill_tokens_per_s=1.0)
    cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                       token_budget=args.budget, max_step_tokens=args.max_step_tokens)
    tokens, secs, n_acc, cpu_s, first_idx = 0, 0.0, 0, 0.0, []
    for w, nw, n in zip(wins, warm_w, per_w):
        end = w["step_ends"][nw + n - 1]
        small = Replay(prof(names[0], BackendRole.SMALL), w["small"], w["window_start"][0], end[0], rep)
        base = Replay(prof(names[1], BackendRole.BASE), w["base"], w["window_start"][1], end[1], rep)
        res = reng.run_trajectory(cfg, w["problem"], small, base)
        first = w["fast_forward_steps"] + nw
        timed = [st for st in res.state.retained_steps if first <= st.index < first + n]
        assert len(timed) == n, (len(timed), n)
        tokens += sum(st.token_count for st in timed)
        n_acc += sum(1 for st in timed if st.producer.value == "Speculator")
        # step cost = the CPU cost of the calls the engine made for it (the
        # trace's per-step call boundaries); with a sampled replay the engine's
        # own clock around score_step would see the sampled time, so it is not used
        lo = w["step_ends"][nw - 1] if nw > 0 else w["window_start"]
        secs += (sum(t for i, t in small.cost.items() if lo[0] <= i < end[0])
                 + sum(t for i, t in base.cost.items() if lo[1] <= i < end[1]))
        cpu_s += small.cpu_s + base.cpu_s
        first_idx.append(first)
    value = round(tokens / secs, 3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (recorded C3 trajectory of this benchmark, bench_data/)",
        "config": bench_config(args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rep.threads, "kind": "port",
                         "sample": (f"reference stepspec engine ({ref_root}) over the recorded "
                                    f"trajectories of this benchmark's {P} windows (timed steps "
                                    f"from indices {first_idx}, {args.warmup} warm-up steps before "
                                    f"the first); every backend call of those steps executes at the "
                                    f"full {names[0]} / {names[1]} shapes on the host cores "
                                    f"(oracle/cpu_replay.py) on a bounded sample per call -- "
                                    f"{rep.sample_text()}; a step's latency = the CPU cost of "
                                    f"its calls")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "loop": {"tokens": tokens, "accepted_fraction": round(n_acc / args.steps, 3),
                 "cpu_seconds_scaled": round(cpu_s, 1),
                 "cpu_seconds_spent": round(rep.wall_s, 1)},
        "wall_s": round(time.perf_counter() - t_start, 1),
    }), flush=True)


def main() -> None:
    if os.environ.get("BENCH_STACK_DUMP_S"):
        import faulthandler

        faulthandler.dump_traceback_later(int(os.environ["BENCH_STACK_DUMP_S"]), repeat=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pair", default="1.5b+32b")
    ap.add_argument("--threshold", type=int, default=7)
    ap.add_argument("--budget", type=int, default=8192)
    ap.add_argument("--max-step-tokens", type=int, default=256)
    ap.add_argument("--problems", type=int, default=64,
                    help="fixed problem set task0000.. (split by id across DP ranks)")
    ap.add_argument("--ff-tokens", type=int, default=-1,
                    help="untimed fast-forward to this many CoT tokens (-1: batch 1 spreads the "
                         "windows over 0.75 * budget, --batch > 1 uses budget / 4)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="CPU work of the cpu_baseline sample (whole timed steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--windows", type=int, default=4,
                    help="batch 1: the timed steps are split over this many problems' windows, "
                         "each after its own fast-forward")
    ap.add_argument("--ref-layer-frac", type=float, default=0.125,
                    help="--impl reference: fraction of each model's layers run per call (scaled back)")
    ap.add_argument("--ref-decode-cap", type=int, default=16,
                    help="--impl reference: decode steps run per generation call (scaled back)")
    ap.add_argument("--dump-trace", default="", help="write the recorded trajectory (reference arm input)")
    ap.add_argument("--trace", default="", help="--impl reference: recorded trajectory to replay")
    ap.add_argument("--verify-template", default="v1", choices=["v1", "v2"],
                    help="v2: prefix-sharing verification prompt (not the reference wording)")
    ap.add_argument("--spec-gamma", type=int, default=0,
                    help="token-level speculation inside base generation (0 = off)")
    ap.add_argument("--batch", type=int, default=1,
                    help="trajectories per GPU run concurrently with batched device passes "
                         "(SURVEY 8f-2; config C5 uses 8); 1 = batch-1 workload")
    ap.add_argument("--sweep", default="",
                    help="C5 threshold sweep, e.g. 3,5,7,9,10: every problem of --problems at every "
                         "threshold plus BaseOnly (problem-id partition over the ranks)")
    ap.add_argument("--mode", default="dp", choices=["dp", "tp"],
                    help="multi-GPU: dp = problem-id partition (C5), tp = base tensor-parallel (C4)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    elif args.sweep:
        run_sweep(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
