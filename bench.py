"""SpecReason inner-loop benchmark (BASELINE.json metric: CoT tokens/s and ms
per reasoning step, draft + verify + fallback).

One *step* is one iteration of the SpecReason thinking loop driven through the
public API (``driver.SpecReasonSession`` over two ``B200Backend``s): the draft
decodes a step, the base scores it in one prefill pass, and on reject the base
regenerates it.  Steps are taken in order from back-to-back configuration-C2
trajectories (1.5B-shape draft + 7B-shape base, random-init bf16, greedy,
threshold 7, 4096-token thinking budget, 64-token synthetic problems); a new
trajectory (new problem) starts whenever one ends.

Reported (one JSON line, rank 0):
  value      CoT tokens / s over the K timed steps, device time (sum of the
             CUDA-event durations of every native call: prefill + decode graph
             + readout), whole job = all ranks' tokens / max rank time
  e2e        the same metric end to end: wall time of the K steps through the
             public API (tokenisation, the Python driver, H2D of ids, D2H of
             results), timed with CUDA events + synchronize around the region
  roofline   the base model's fallback decode step graph (the dominant cost):
             algorithmic bytes (weights + KV read per token) / its
             CUDA-event time, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the CPU oracle (fp32, torch on the host cores) on a bounded
             sample, layer-sliced and extrapolated by weight bytes
Multi-GPU: one process per GPU (torchrun), independent problems per rank (no
collective on the data path): scaling "weak".
``--impl reference`` times the reference loop on the host CPU instead (rank 0).
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
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


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
    """Endless sequence of SpecReason steps over back-to-back trajectories."""

    def __init__(self, small, base, config, problems, vocab) -> None:
        from paper_2504_07891_b200.driver import SpecReasonSession

        self.cls = SpecReasonSession
        self.small, self.base, self.config = small, base, config
        self.problems = problems
        self.vocab = vocab
        self.k = 0
        self.trajectories = 0
        self.session = None
        self._new()

    def _new(self) -> None:
        seed = self.problems[self.k % len(self.problems)]
        self.k += 1
        self.session = self.cls(self.config, self.vocab.problem(64, seed), self.small, self.base)
        self.trajectories += 1

    def step(self):
        while True:
            out = self.session.step()
            if out is not None:
                return out
            self._new()


def run_ours(args) -> None:
    from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
    from paper_2504_07891_b200.backend import build_pair
    from paper_2504_07891_b200.shapes import PAIRS, get_spec
    from paper_2504_07891_b200.vocab import shared_vocab

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    base_tp = None
    if args.mode == "tp":  # config C4: base sharded over the ranks, one shared trajectory
        from paper_2504_07891_b200.backend import TensorParallel

        base_tp = TensorParallel.from_dist() if dist is not None else TensorParallel.single()
    extra = {"n_streams": 2 * args.batch + 2, "max_tokens": 1024} if args.batch > 1 else {}
    small, base = build_pair(args.pair, seed=args.seed, max_ctx=args.budget + 512,
                             threshold=args.threshold, base_tp=base_tp, **extra)
    base.verify_template = args.verify_template
    if args.spec_gamma > 0:  # SpecReason+Decode: the draft proposes tokens inside base fallback
        base.attach_speculator(small, gamma=args.spec_gamma)
    vocab = shared_vocab(get_spec(PAIRS[args.pair][0]).vocab_text)
    cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                       token_budget=args.budget, max_step_tokens=args.max_step_tokens)
    # DP: independent problems per rank; TP: every rank drives the same one
    problems = [(0 if args.mode == "tp" else rank) * 1000 + i for i in range(64)]
    sched = None
    if args.batch > 1:  # B trajectories, each on its own thread, batched device passes
        from paper_2504_07891_b200.batching import BatchScheduler

        sched = BatchScheduler(small, base)
        srcs = [StepSource(sched.small, sched.base, cfg, problems[k::args.batch], vocab)
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
        run_steps(max(1, -(-args.warmup // args.batch)))
    else:
        src = StepSource(small, base, cfg, problems, vocab)
        for _ in range(args.warmup):
            src.step()

    stream = torch.cuda.current_stream()
    s0 = (small.engine.stats.snapshot(), base.engine.stats.snapshot())
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outcomes = []
    with ClockSampler(local) as clocks:
        e0.record(stream)
        if sched is not None:
            outcomes = run_steps(per)
        else:
            for _ in range(args.steps):
                outcomes.append(src.step())
        e1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    wall_ms = e0.elapsed_time(e1)
    n_steps = len(outcomes)  # --batch B runs ceil(steps / B) steps on each trajectory
    ds = small.engine.stats.minus(s0[0])
    db = base.engine.stats.minus(s0[1])

    tokens = sum(o.step.token_count for o in outcomes)
    dev_ms = ds.prefill_ms + ds.decode_ms + db.prefill_ms + db.decode_ms
    lat = [o.step.latency for o in outcomes]
    n_spec = sum(1 for o in outcomes if o.action.value == "AcceptedSpeculation")

    tot_tokens = _reduce_sum(dist, tokens) if args.mode == "dp" else tokens
    max_dev_ms = _reduce_max(dist, dev_ms)
    max_wall_ms = _reduce_max(dist, wall_ms)
    peaks = _peaks()
    ach = db.decode_bytes / (db.decode_ms * 1e-3) / 1e9 if db.decode_ms > 0 else 0.0

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
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
        "data": "synthetic (random-init weights, seeded 64-word problems)",
        "config": {"workload": WORKLOADS[args.pair].replace("batch 1", f"batch {args.batch}"), "pair": args.pair, "threshold": args.threshold,
                   "verify_template": args.verify_template, "spec_gamma": args.spec_gamma,
                   "token_budget": args.budget, "max_step_tokens": args.max_step_tokens,
                   "batch": args.batch, "parallelism": (f"dp{world} (independent problems per GPU"
                                               + (f", {args.batch} concurrent trajectories per GPU "
                                                  "sharing batched device passes)" if args.batch > 1 else ")")
                                               if args.mode == "dp" else
                                               f"tp{world} (base sharded, NCCL all-reduce; draft replicated)"),
                   "l2": "weights (17 GB) exceed L2 (126 MB): no flush needed"},
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
                 "trajectories": src.trajectories,
                 "draft_decode_ms_per_token": round(ds.decode_ms / max(1, ds.decode_tokens), 4),
                 "base_decode_ms_per_token": round(db.decode_ms / max(1, db.decode_tokens), 4),
                 "base_prefill_tokens": db.prefill_tokens, "base_prefill_ms": round(db.prefill_ms, 2)},
        "roofline": {"kernel": "decode_mk_kernel (persistent weight-streaming decode, base model "
                               "fallback steps): algorithmic bytes = 2*(P_body+P_head) + (C+1)*kvB "
                               "per token (SURVEY 8d) / CUDA-event decode time",
                     "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                     "peak_source": peaks["src"],
                     # ncu --set full of the same kernel (7B base, C~2K): DRAM bytes
                     # read+written per decoded token, vs the algorithmic bytes
                     "traffic": 14.271e9 if args.pair == "1.5b+7b" else None,
                     "traffic_unit": "bytes/token (profiles/r01_ncu_decode_mk_qwen2.5-7b_summary.txt)",
                     "algorithmic_bytes_per_token": round(db.decode_bytes / max(1, db.decode_tokens)),
                     "draft_decode_GBps": round(ds.decode_bytes / (ds.decode_ms * 1e-3) / 1e9, 1)
                     if ds.decode_ms > 0 else None},
        "gpu_launches": ds.launches + db.launches,
        **({"batching": {"trajectories_in_flight": args.batch,
                         "device_passes": len(sched.batches),
                         "mean_requests_per_pass": round(sum(sched.batches) / max(1, len(sched.batches)), 2)}}
           if sched is not None else {}),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, outcomes_stats=(ds, db, tokens, n_steps))
    print(json.dumps(result), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ----------------------------------------------------------------- CPU arm --
def _cpu_costs(args, layers: int):
    """Per-token CPU cost (s) of decode and prefill for both models, measured
    on ``layers``-layer slices of the real shapes and extrapolated to the full
    depth by weight bytes (CPU decode is memory-bound)."""
    from oracle.ref_model import RefModel
    from paper_2504_07891_b200.shapes import PAIRS, get_spec, make_weights

    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    out = {}
    for name in PAIRS[args.pair]:
        spec = get_spec(name)
        keep = list(range(min(layers, spec.n_layers)))
        w = make_weights(spec, args.seed, device="cpu", layers=keep)
        m = RefModel(spec, w, max_pos=4096 + 1024, layers=keep)
        del w
        body_per_layer = (spec.body_params() - spec.d_model) / spec.n_layers
        full = spec.body_params() + spec.head_params()
        sliced = body_per_layer * len(keep) + spec.head_params()
        scale = full / sliced
        g = torch.Generator().manual_seed(1)
        ids = torch.randint(16, 4000, (512,), generator=g).tolist()
        cache = m.new_cache()
        t0 = time.perf_counter()
        m.forward(cache, ids[:80])
        prefill_s = (time.perf_counter() - t0) / 80 * scale
        t0 = time.perf_counter()
        n_dec = 6
        for t in ids[80:80 + n_dec]:
            m.forward(cache, [t])
        decode_s = (time.perf_counter() - t0) / n_dec * scale
        out[name] = {"decode_s_per_token": decode_s, "prefill_s_per_token": prefill_s,
                     "scale": round(scale, 3)}
        del m
    return out, threads


def cpu_baseline(args, outcomes_stats) -> dict:
    """Oracle on the host cores for the same step mix as the timed GPU steps."""
    ds, db, tokens, steps = outcomes_stats
    costs, threads = _cpu_costs(args, args.ref_layers)
    from paper_2504_07891_b200.shapes import PAIRS

    dn, bn = PAIRS[args.pair]
    cpu_s = (ds.prefill_tokens * costs[dn]["prefill_s_per_token"]
             + (ds.decode_tokens + ds.calls) * costs[dn]["decode_s_per_token"]
             + db.prefill_tokens * costs[bn]["prefill_s_per_token"]
             + db.decode_tokens * costs[bn]["decode_s_per_token"])
    return {"value": round(tokens / cpu_s, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"fp32 torch oracle on {args.ref_layers}-layer slices of both models "
                      f"(80-token prefill, 6 decode tokens each), extrapolated to full depth by "
                      f"weight bytes and applied to the timed steps' token mix",
            "ms_per_step": round(1e3 * cpu_s / steps, 1), "per_token_costs": costs}


def run_reference(args) -> None:
    """Reference arm: the reference's loop on the host CPU (oracle port for
    the model arithmetic; the unmodified reference engine when installed in
    baseline/_ref).  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ref_path = ROOT / "baseline" / "_ref"
    engine_kind = "this repo's driver (reference not installed)"
    run_traj = None
    if (ref_path / "stepspec").exists():
        sys.path.insert(0, str(ref_path))
        try:
            import stepspec  # noqa: F401
            from stepspec import engine as reng

            engine_kind = "reference stepspec engine (baseline/_ref)"
            run_traj = reng
        except Exception:  # noqa: BLE001
            run_traj = None
    costs, threads = _cpu_costs(args, args.ref_layers)
    # the reference loop on the CPU oracle: a tiny-pair trajectory gives the
    # step mix (tokens / calls per step); costs are the C2 shapes' per-token costs
    from oracle.ref_engine import oracle_backend
    from paper_2504_07891_b200 import AcceptanceThreshold, EngineConfig
    from paper_2504_07891_b200.domain import BackendRole
    from paper_2504_07891_b200.host import reference_types
    from paper_2504_07891_b200.shapes import PAIRS
    from paper_2504_07891_b200.vocab import shared_vocab

    T = reference_types(sys.modules["stepspec"]) if run_traj is not None else None
    small = oracle_backend("tiny-draft", BackendRole.SMALL, types=T, record=True)
    base = oracle_backend("tiny-base", BackendRole.BASE, types=T, record=True,
                          threshold=args.threshold)
    v = shared_vocab(4096)
    if run_traj is not None:
        from stepspec.core import AcceptanceThreshold as RT
        from stepspec.core import EngineConfig as RC

        cfg = RC(threshold=RT(args.threshold), temperature=0.0, token_budget=args.budget,
                 max_step_tokens=args.max_step_tokens)
    else:
        cfg = EngineConfig(threshold=AcceptanceThreshold(args.threshold), temperature=0.0,
                           token_budget=args.budget, max_step_tokens=args.max_step_tokens)
    dn, bn = PAIRS[args.pair]
    per_step = []  # (CoT tokens, CPU seconds at the C2 shapes)
    t_start = time.perf_counter()
    p = 0
    while len(per_step) < args.warmup + args.steps:
        small.calls.clear()
        base.calls.clear()
        prob = v.problem(64, p)
        p += 1
        if run_traj is not None:
            res = run_traj.run_trajectory(cfg, prob, small, base)
        else:
            from paper_2504_07891_b200.driver import run_trajectory

            res = run_trajectory(cfg, prob, small, base)
        calls = sorted([("small", c) for c in small.calls] + [("base", c) for c in base.calls],
                       key=lambda x: x[1]["seq"])
        # a step starts at each draft call; the answer (last base call) is not a step
        groups, cur = [], None
        for who, c in calls:
            if who == "small":
                cur = [c["fresh"] * costs[dn]["prefill_s_per_token"]
                       + len(c["gen_ids"]) * costs[dn]["decode_s_per_token"]]
                groups.append(cur)
            elif cur is not None:
                if c["kind"] == "score":
                    cur.append(c["fresh"] * costs[bn]["prefill_s_per_token"])
                else:
                    cur.append(c["fresh"] * costs[bn]["prefill_s_per_token"]
                               + len(c["gen_ids"]) * costs[bn]["decode_s_per_token"])
        for st, g in zip(res.state.retained_steps, groups):
            per_step.append((st.token_count, sum(g)))
    timed = per_step[args.warmup:]
    tokens = sum(t for t, _ in timed)
    secs = sum(s for _, s in timed)
    value = round(tokens / secs, 3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / len(timed), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.pair].replace("batch 1", f"batch {args.batch}"), "pair": args.pair,
                                        "threshold": args.threshold, "token_budget": args.budget},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{engine_kind} driving the CPU oracle; per-token CPU costs of "
                                   f"the C2 shapes measured on {args.ref_layers}-layer slices and "
                                   f"extrapolated by weight bytes, applied to each step's tokens",
                         "per_token_costs": costs},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_start, 1),
    }), flush=True)


def main() -> None:
    if os.environ.get("BENCH_STACK_DUMP_S"):
        import faulthandler

        faulthandler.dump_traceback_later(int(os.environ["BENCH_STACK_DUMP_S"]), repeat=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # the loop's step mix (draft steps accepted or regenerated) varies a lot
    # between random-init trajectories (one C2 trajectory is ~130 steps): 480
    # steps average over several of them and still run in about a minute
    ap.add_argument("--steps", type=int, default=480)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pair", default="1.5b+7b")
    ap.add_argument("--threshold", type=int, default=7)
    ap.add_argument("--budget", type=int, default=4096)
    ap.add_argument("--max-step-tokens", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ref-layers", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verify-template", default="v1", choices=["v1", "v2"],
                    help="v2: prefix-sharing verification prompt (not the reference wording)")
    ap.add_argument("--spec-gamma", type=int, default=0,
                    help="token-level speculation inside base generation (0 = off)")
    ap.add_argument("--batch", type=int, default=1,
                    help="trajectories per GPU run concurrently with batched device passes "
                         "(SURVEY 8f-2; config C5 uses 8); 1 = the C2 batch-1 workload")
    ap.add_argument("--mode", default="dp", choices=["dp", "tp"],
                    help="multi-GPU: dp = independent problems per rank (C5), "
                         "tp = base model tensor-parallel over the ranks (C4)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
