"""CPU cost replay of recorded backend calls -- TEST / BASELINE INFRASTRUCTURE
ONLY (used by ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference``
arm; the product never imports it).

What it measures: the wall time the host cores need to execute, at the full
model shape and depth, the arithmetic each recorded backend call implies --
a generation call prefills its fresh prompt suffix at its real context
position and then decodes its tokens one by one, each decode step reading
every weight and the K/V of the whole context; a scoring call prefills its
fresh rows and reads the judge position's logits.  This is the oracle's
computation (``ref_model.RefModel``: RMSNorm, GQA attention with RoPE over
the cached context, SwiGLU, LM head) with its bf16 storage points, executed
by torch on the CPU with bf16 matmuls accumulating in fp32 (the oneDNN /
AMX path -- the fastest exact-input CPU formulation, so the baseline is not
handicapped by upcasting weights).

Cost-faithful, value-free: the time of these kernels does not depend on the
numbers, so one random layer of weights is reused for all ``n_layers``
(every layer still streams its full weight bytes from DRAM: a layer is ~1 GB
at the 32B shape, far beyond the last-level cache) and the context's K/V are
random values at the recorded length.  The tokens and scores themselves come
from the recorded (device) trajectory; the CPU replay only prices them.
"""

from __future__ import annotations

import math
import os
import time

import torch

from paper_2504_07891_b200.shapes import ModelSpec, rope_table

PREFILL_CHUNK = 256


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


class CpuModel:
    """One model's per-call CPU executor (see module doc)."""

    def __init__(self, spec: ModelSpec, max_ctx: int, seed: int = 0) -> None:
        self.spec = spec
        d, hd = spec.d_model, spec.head_dim
        g = torch.Generator().manual_seed(seed)

        def rnd(rows, cols, std):
            # tile a random block: cheap to create, every byte distinct in DRAM
            blk = (torch.randn(min(rows, 2048), cols, generator=g) * std).to(torch.bfloat16)
            reps = -(-rows // blk.shape[0])
            return blk.repeat(reps, 1)[:rows].contiguous()

        self.wqkv = rnd(spec.qkv_rows, d, d ** -0.5)
        self.bqkv = (torch.randn(spec.qkv_rows, generator=g) * 0.02).to(torch.bfloat16)
        self.wo = rnd(d, spec.q_dim, spec.q_dim ** -0.5)
        self.wgu = rnd(2 * spec.d_ffn, d, d ** -0.5)
        self.wd = rnd(d, spec.d_ffn, spec.d_ffn ** -0.5)
        self.lm_head = rnd(spec.vocab_rows, d, d ** -0.5)
        self.embed = rnd(4096, d, 1.0)
        self.kv_k = (torch.randn(max_ctx, spec.n_kv_heads, hd, generator=g)).to(torch.bfloat16)
        self.kv_v = (torch.randn(max_ctx, spec.n_kv_heads, hd, generator=g)).to(torch.bfloat16)
        tab = rope_table(spec, max_ctx)
        self.cos, self.sin = tab[..., 0], tab[..., 1]
        self.max_ctx = max_ctx

    def _norm(self, h: torch.Tensor) -> torch.Tensor:
        ms = (h * h).mean(dim=-1, keepdim=True)
        return (h * torch.rsqrt(ms + self.spec.rms_eps)).to(torch.bfloat16)

    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        half = x.shape[-1] // 2
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    @torch.no_grad()
    def forward(self, start: int, n: int, logits: bool = True, layers: int | None = None) -> int:
        """``n`` new positions at ``start``.. through every layer (or the
        first ``layers`` of them: a layer sample) with context ``start``
        cached, then the LM head of the last row; returns argmax."""
        spec = self.spec
        if start + n > self.max_ctx:
            raise ValueError("context exceeds the replay cache")
        H, KV, hd, G = spec.n_heads, spec.n_kv_heads, spec.head_dim, spec.group
        pos = torch.arange(start, start + n)
        h = self.embed[pos % self.embed.shape[0]].float()
        scale = 1.0 / math.sqrt(hd)
        T = start + n
        for _ in range(spec.n_layers if layers is None else layers):
            x = self._norm(h)
            qkv = (x @ self.wqkv.T + self.bqkv).float()
            q = self._rope(qkv[:, : spec.q_dim].view(n, H, hd), pos).to(torch.bfloat16)
            k = self._rope(qkv[:, spec.q_dim: spec.q_dim + spec.kv_dim].view(n, KV, hd), pos)
            self.kv_k[start:T] = k.to(torch.bfloat16)
            self.kv_v[start:T] = qkv[:, spec.q_dim + spec.kv_dim:].view(n, KV, hd).to(torch.bfloat16)
            Kx = self.kv_k[:T].permute(1, 2, 0)                       # [KV, hd, T]
            Vx = self.kv_v[:T].permute(1, 0, 2)                       # [KV, T, hd]
            qg = q.view(n, KV, G, hd).permute(1, 0, 2, 3).reshape(KV, n * G, hd)
            s = torch.bmm(qg, Kx).float() * scale                    # [KV, n*G, T]
            if n > 1:
                mask = torch.arange(T)[None, :] > pos[:, None]
                s = s.view(KV, n, G, T).masked_fill(mask[None, :, None, :], float("-inf")).view(KV, n * G, T)
            p = torch.softmax(s, dim=-1).to(torch.bfloat16)
            o = torch.bmm(p, Vx).view(KV, n, G, hd).permute(1, 0, 2, 3).reshape(n, spec.q_dim)
            h = h + (o @ self.wo.T).float()
            x2 = self._norm(h)
            gu = (x2 @ self.wgu.T).float().view(n, -1, 2, 16)
            act = (torch.nn.functional.silu(gu[:, :, 0]) * gu[:, :, 1]).reshape(n, -1)
            h = h + (act.to(torch.bfloat16) @ self.wd.T).float()
        if not logits:
            return -1
        lg = self._norm(h[-1:]) @ self.lm_head.T
        return int(lg.float().argmax())

    def generate(self, start: int, n_fresh: int, n_gen: int, layers: int | None = None,
                 decode_cap: int | None = None) -> float:
        """A generation call: prefill ``n_fresh`` rows (chunked), then
        ``n_gen - 1`` decode steps (the first token comes from the prefill).
        Returns the call's seconds; with a sample (``layers`` of the model's
        layers, at most ``decode_cap`` decode steps spread over the call) the
        sampled time is scaled back: layer parts by n_layers / layers (every
        layer streams the same bytes: one random layer is reused), decode by
        (n_gen - 1) / steps run.  The LM head is always run once per token."""
        L = self.spec.n_layers
        lf = 1.0 if layers is None else L / layers
        t_body = t_head = 0.0
        c0 = 0
        while c0 < n_fresh:
            m = min(PREFILL_CHUNK, n_fresh - c0)
            t0 = time.perf_counter()
            self.forward(start + c0, m, logits=False, layers=layers)
            t_body += time.perf_counter() - t0
            c0 += m
        t0 = time.perf_counter()
        self.forward(start + n_fresh - 1, 1, logits=True, layers=0)  # LM head of the last row
        t_head += time.perf_counter() - t0
        total = t_body * lf + t_head
        nd = max(0, n_gen - 1)
        run = nd if decode_cap is None else min(nd, decode_cap)
        if run:
            t0 = time.perf_counter()
            for j in range(run):
                i = j * nd // run  # spread over the call's positions
                self.forward(start + n_fresh + i, 1, layers=layers)
            td = time.perf_counter() - t0
            # each sampled step = body (layer-sampled) + head: scale the body only
            head1 = t_head
            body_per = max(0.0, td / run - head1)
            total += nd * (body_per * lf + head1)
        return total

    def score(self, start: int, n_fresh: int, layers: int | None = None) -> float:
        """A scoring call: prefill the fresh rows, read the last row's logits."""
        return self.generate(start, n_fresh, 1, layers=layers)


class CpuReplay:
    """Executes recorded call descriptors ``{"model", "kind", "start",
    "fresh", "n_gen"}`` on the CPU models of a pair; returns seconds.

    ``layer_frac`` / ``decode_cap`` bound the work per call (a sample of the
    layers and of the decode steps, scaled back as ``CpuModel.generate``
    states); ``None`` executes every layer and token."""

    def __init__(self, specs: dict[str, ModelSpec], max_ctx: int, threads: int | None = None,
                 layer_frac: float | None = None, decode_cap: int | None = None) -> None:
        self.threads = threads or host_threads()
        torch.set_num_threads(self.threads)
        self.models = {k: CpuModel(s, max_ctx) for k, s in specs.items()}
        self.layers = {k: (None if layer_frac is None else max(1, round(s.n_layers * layer_frac)))
                       for k, s in specs.items()}
        self.decode_cap = decode_cap
        self.wall_s = 0.0  # host seconds actually spent

    def sample_text(self) -> str:
        if all(v is None for v in self.layers.values()) and self.decode_cap is None:
            return "every layer and token"
        parts = [f"{k}: {v} of {self.models[k].spec.n_layers} layers" for k, v in self.layers.items()]
        return ("; ".join(parts) + (f"; <= {self.decode_cap} decode steps per call" if self.decode_cap else "")
                + " (scaled back per call)")

    def warm(self) -> None:
        for m in self.models.values():
            m.forward(0, 8)
            m.forward(8, 1)

    def run(self, call: dict) -> float:
        m = self.models[call["model"]]
        lay = self.layers[call["model"]]
        t0 = time.perf_counter()
        if call["kind"] == "score":
            t = m.score(call["start"], call["fresh"], layers=lay)
            if call.get("catchup"):  # the generation stream's rows of the same pass,
                # which the reference's own fallback call would prefill instead
                t += m.generate(call["catchup_start"], call["catchup"], 0, layers=lay)
        else:
            t = m.generate(call["start"], call["fresh"], call["n_gen"], layers=lay,
                           decode_cap=self.decode_cap)
        self.wall_s += time.perf_counter() - t0
        return t
