"""CPU fp32 restatement of the decoder arithmetic -- TEST INFRASTRUCTURE ONLY.

This is the parity oracle for the sm_100a kernels.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product path
(``paper_2504_07891_b200``) never does.

What it restates: the reference delegates all model arithmetic to an external
vLLM server (``backends/http.py:63-94``; vLLM 0.8.2 per ``PAPER.md:210``, not
pinned in ``pyproject.toml:10-13`` and not vendored), so there is no
reference source for the math.  The oracle is a plain Qwen2-style decoder
(RMSNorm, GQA attention with q/k/v bias and rotate-half RoPE, SwiGLU, untied
LM head), written from the public architecture, in fp32 on the CPU.

Storage points: the GPU keeps activations that feed a matmul, the K/V cache
and the attention output in bf16, and the residual stream in fp32.  The oracle
rounds to bf16 at exactly those points (``_r``) and accumulates everything in
fp32, so GPU-vs-oracle differences come only from summation order and rare
bf16 rounding flips.  ``exact_fp32=True`` disables the rounding (a pure fp32
reference) for tolerance studies.

Parity of the surrounding control flow (tokens, steps, scores, accept/reject)
is pinned against the reference's own tests and engine: see
``tests/test_reference_pins.py`` and ``tests/golden/make_golden.py``.
"""

from __future__ import annotations

import math

import torch

from paper_2504_07891_b200.shapes import ModelSpec, gu_split, rope_table


def _r(x: torch.Tensor, on: bool) -> torch.Tensor:
    return x.to(torch.bfloat16).to(x.dtype) if on else x


class RefModel:
    """Teacher-forced / incremental fp32 forward over a per-stream KV cache."""

    def __init__(self, spec: ModelSpec, weights: dict[str, torch.Tensor],
                 max_pos: int = 32768, exact_fp32: bool = False,
                 layers: list[int] | None = None, dtype: torch.dtype = torch.float32) -> None:
        """``dtype=torch.float64`` keeps the same bf16 storage points but
        computes in double: the pair (fp32, fp64) measures the intrinsic
        summation-order noise floor any fp32 implementation has."""
        self.spec = spec
        self.round = not exact_fp32
        self.dtype = dtype
        f = lambda t: t.to(dtype).contiguous()  # noqa: E731
        self.embed = f(weights["embed"])
        self.ln_f = f(weights["ln_f"])
        self.lm_head = f(weights["lm_head"])
        self.layers = []
        ids = layers if layers is not None else list(range(spec.n_layers))
        for i in ids:
            p = f"layers.{i}."
            gate, up = gu_split(weights[p + "wgu"])
            self.layers.append({
                "ln1": f(weights[p + "ln1"]), "wqkv": f(weights[p + "wqkv"]),
                "bqkv": f(weights[p + "bqkv"]), "wo": f(weights[p + "wo"]),
                "ln2": f(weights[p + "ln2"]), "wg": f(gate), "wu": f(up),
                "wd": f(weights[p + "wd"]),
            })
        tab = rope_table(spec, max_pos).to(dtype)
        self.cos, self.sin = tab[..., 0], tab[..., 1]

    # -- cache -----------------------------------------------------------
    def new_cache(self) -> dict:
        return {"k": [None] * len(self.layers), "v": [None] * len(self.layers), "len": 0}

    @staticmethod
    def truncate(cache: dict, keep: int) -> None:
        if keep < cache["len"]:
            cache["k"] = [None if k is None else k[:keep] for k in cache["k"]]
            cache["v"] = [None if v is None else v[:keep] for v in cache["v"]]
            cache["len"] = keep

    # -- pieces ----------------------------------------------------------
    def _norm(self, h: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        ms = (h * h).mean(dim=-1, keepdim=True)
        return _r(h * torch.rsqrt(ms + self.spec.rms_eps) * w, self.round)

    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        # x [n, heads, hd]; rotate-half pairs (i, i + hd/2)
        half = x.shape[-1] // 2
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def forward(self, cache: dict, ids: list[int], last_only: bool = True,
                hidden_only: bool = False) -> torch.Tensor:
        """Append ``ids`` at positions cache.len.. and return fp32 logits of
        the last position ([V]) or of every new position ([n, V])."""
        spec, rd = self.spec, self.round
        n = len(ids)
        start = cache["len"]
        pos = torch.arange(start, start + n)
        h = self.embed[torch.tensor(ids, dtype=torch.long)].clone()
        hd, H, KV = spec.head_dim, spec.n_heads, spec.n_kv_heads
        scale = 1.0 / math.sqrt(hd)
        for li, L in enumerate(self.layers):
            x = self._norm(h, L["ln1"])
            qkv = x @ L["wqkv"].T + L["bqkv"]
            q = qkv[:, : spec.q_dim].view(n, H, hd)
            k = qkv[:, spec.q_dim: spec.q_dim + spec.kv_dim].view(n, KV, hd)
            v = qkv[:, spec.q_dim + spec.kv_dim:].view(n, KV, hd)
            q = _r(self._rope(q, pos), rd)
            k = _r(self._rope(k, pos), rd)
            v = _r(v, rd)
            pk, pv = cache["k"][li], cache["v"][li]
            K = k if pk is None else torch.cat([pk, k], 0)
            V = v if pv is None else torch.cat([pv, v], 0)
            cache["k"][li], cache["v"][li] = K, V
            T = K.shape[0]
            # scores [H, n, T]; GQA: q head j uses kv head j // group
            Kx = K.repeat_interleave(spec.group, dim=1).permute(1, 2, 0)  # [H, hd, T]
            Vx = V.repeat_interleave(spec.group, dim=1).permute(1, 0, 2)  # [H, T, hd]
            s = torch.bmm(q.permute(1, 0, 2), Kx) * scale
            mask = torch.arange(T)[None, :] > (pos[:, None])
            s = s.masked_fill(mask[None], float("-inf"))
            p = torch.softmax(s, dim=-1)
            o = torch.bmm(p, Vx).permute(1, 0, 2).reshape(n, spec.q_dim)
            o = _r(o, rd)
            h = h + o @ L["wo"].T
            x2 = self._norm(h, L["ln2"])
            g = x2 @ L["wg"].T
            u = x2 @ L["wu"].T
            a = _r(torch.nn.functional.silu(g) * u, rd)
            h = h + a @ L["wd"].T
        cache["len"] = start + n
        hf = h[-1:] if last_only else h
        xf = self._norm(hf, self.ln_f)
        if hidden_only:
            return xf
        logits = xf @ self.lm_head.T
        return logits[0] if last_only else logits


def masked(logits: torch.Tensor, n_text: int) -> torch.Tensor:
    """Padding rows (>= n_text) can never be chosen."""
    if logits.shape[-1] > n_text:
        logits = logits.clone()
        logits[..., n_text:] = float("-inf")
    return logits


def argmax_margin(logits: torch.Tensor) -> tuple[int, float]:
    """(greedy id, top1 - top2): first index wins exact ties."""
    top = torch.topk(logits, 2)
    return int(torch.argmax(logits)), float(top.values[0] - top.values[1])
