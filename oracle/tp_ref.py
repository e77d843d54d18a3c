"""Tensor-parallel restatement of the oracle forward -- TEST INFRASTRUCTURE ONLY.

The decomposition the device runtime uses for the base model at TP > 1
(Megatron-style), written with torch.distributed collectives so
that a world-size-2 gloo run on the CPU checks it against the unsharded
oracle (``ref_model.RefModel``):

  per layer   x = RMSNorm(h)                       (replicated)
              q, k, v = x @ Wqkv_r^T + b_r          (this rank's heads)
              o_r = attention(q, k, v) @ Wo_r^T     (row-parallel partial)
              h  += all_reduce(o_r)
              a_r = silu(x2 @ Wg_r^T) * (x2 @ Wu_r^T)   (this rank's ffn units)
              h  += all_reduce(a_r @ Wd_r^T)
  LM head     logits = all_gather(RMSNorm(h) @ Wlm_r^T)  (vocab-parallel)

Storage points (bf16 rounding) are the oracle's.  Weights are the shards of
``shapes.shard_weights``, the function the device path loads.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from paper_2504_07891_b200.shapes import ModelSpec, gu_split, rope_table, shard_weights, tp_spec

from .ref_model import _r


def tp_forward_logits(spec: ModelSpec, full: dict[str, torch.Tensor], ids: list[int],
                      rank: int, world: int) -> torch.Tensor:
    """[n, V] fp32 logits of every position of `ids`, computed by rank `rank`
    of `world` (gloo) with this rank's shard only."""
    rs = tp_spec(spec, rank, world)
    w = {k: v.float() for k, v in shard_weights(full, spec, rank, world).items()}
    n = len(ids)
    hd, H, KV = spec.head_dim, rs.n_heads, rs.n_kv_heads
    group = spec.n_heads // spec.n_kv_heads
    tab = rope_table(spec, n + 1)
    cos, sin = tab[:n, :, 0], tab[:n, :, 1]
    pos = torch.arange(n)

    def norm(x, g):
        ms = (x * x).mean(dim=-1, keepdim=True)
        return _r(x * torch.rsqrt(ms + spec.rms_eps) * g, True)

    def rope(x):
        half = hd // 2
        c, s = cos[:, None, :], sin[:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    h = w["embed"][torch.tensor(ids, dtype=torch.long)].clone()
    for i in range(spec.n_layers):
        p = f"layers.{i}."
        x = norm(h, w[p + "ln1"])
        qkv = x @ w[p + "wqkv"].T + w[p + "bqkv"]
        q = _r(rope(qkv[:, : H * hd].view(n, H, hd)), True)
        k = _r(rope(qkv[:, H * hd:(H + KV) * hd].view(n, KV, hd)), True)
        v = _r(qkv[:, (H + KV) * hd:].view(n, KV, hd), True)
        Kx = k.repeat_interleave(group, dim=1).permute(1, 2, 0)
        Vx = v.repeat_interleave(group, dim=1).permute(1, 0, 2)
        s = torch.bmm(q.permute(1, 0, 2), Kx) / math.sqrt(hd)
        s = s.masked_fill((torch.arange(n)[None, :] > pos[:, None])[None], float("-inf"))
        o = _r(torch.bmm(torch.softmax(s, -1), Vx).permute(1, 0, 2).reshape(n, H * hd), True)
        part = o @ w[p + "wo"].T
        dist.all_reduce(part)
        h = h + part
        x2 = norm(h, w[p + "ln2"])
        gate, up = gu_split(w[p + "wgu"])
        a = _r(torch.nn.functional.silu(x2 @ gate.T) * (x2 @ up.T), True)
        part = a @ w[p + "wd"].T
        dist.all_reduce(part)
        h = h + part
    local = norm(h, w["ln_f"]) @ w["lm_head"].T
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts, dim=-1)
