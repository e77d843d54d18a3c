"""Model shapes and seeded random-init weights (Qwen2-style decoders).

The reference names the model pairs but carries no weights or shapes
(``PAPER.md:204``); SURVEY.md §8 fixes the public model-card shapes used
here.  Weights are N(0, 0.02) rounded to bf16 once; norms are 1; q/k/v carry
a bias (Qwen2).  Every tensor has its own keyed seed, so any subset (e.g. one
layer for a CPU parity slice) can be regenerated independently.

The judge circuit
-----------------
A random-init base model essentially never ranks a digit token inside its
top-10 at the end of the verify prompt, so every score would be a parse
failure (-> reject).  To exercise both branches of the loop the base model
carries a small, documented "judge circuit" in its weights only:

* the embedding row of the judge-cue word ``"0-9:"`` (the verify template's
  last word, ``prompts.py:66``) is ``cue_gain * sqrt(d) * u`` for a fixed unit
  vector ``u``, so the residual stream at that position points along ``u``;
* each digit's LM-head row gets ``(digit_gain + judge_offsets[j]) * u / sqrt(d)``
  added, lifting all ten digits into the top-10 *only* at the cue position;
  the random part of those rows (orthogonalised against ``u``) decides which
  digit wins from the context-dependent remainder of the hidden state;
* ``judge_offsets`` equalise the ten digits' mean logit over synthetic verify
  prompts (without them the context-independent part of the cue's hidden
  state pins the score to one or two digits).  They are measured once per
  (model, seed) by ``tools/calibrate_judge.py`` and stored below; the first
  padding row of the LM head is a probe ``u / sqrt(d)`` that reads the cue
  alignment the calibration needs (padding rows are never produced).

* the **probe head** (``probe_gain`` > 0, bench base models): in the last
  layer, q head 0 reads the cue direction (its q rows are ``u`` placed on
  the RoPE pairs of ``probe_pairs``) and kv head 0's keys are a constant
  bias phased so that, after RoPE, the score peaks at distance
  ``probe_offset`` = 36 -- the last word of the candidate step (the verify
  template's tail after the candidate is 35 words).  The head's output
  columns of W_o are scaled by ``probe_gain``.  So the cue position copies
  the value vector of the candidate's last word, and the digit rows' random
  part turns it into the score: consecutive steps of one trajectory get
  nearly independent scores (``tools/calibrate_judge.py`` reports the
  consecutive-equal rate, ~0.15 against 0.1 for independent draws) instead
  of the long-range context deciding one score for a whole trajectory.

The successor circuit
---------------------
A greedy random-init decoder falls into short loops: its final hidden state
is ~85% one direction common to all positions, so a few "hub" tokens win
every argmax, and a step that loops without a boundary word runs to
``max_step_tokens`` (measured: 23-69% of C2 draft steps capped at 256).  The
bench models therefore carry a successor circuit: embeddings are N(0, 1)
(``embed_std``) so the current token stays visible in the last residual,
and every ordinary word's LM-head row gets ``succ_gain`` times the unit
embedding of its predecessor under a seeded permutation of the ordinary ids
(``successor_perm``, keyed by the vocabulary, so draft and base share it).
Greedy text then walks the permutation (~90% of draft tokens, ~99% of base
tokens follow it) instead of looping, boundary words (1 in 24 ids) end steps
at ~24 tokens as SURVEY §7.1 asks (mean 24, p90 ~55, none capped), and a
draft and its base agree on most tokens, as a real distilled pair does.

All of it is plain weight values: the kernels contain no special case.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from .pricing import derive_seed
from .vocab import DIGIT_IDS, JUDGE_CUE_ID


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ffn: int
    vocab_rows: int          # LM-head / embedding rows (may include padding)
    vocab_text: int          # ids that are real words (argmax masks the rest)
    head_dim: int = 128
    rope_theta: float = 1_000_000.0
    rms_eps: float = 1e-6
    init_std: float = 0.0    # 0 -> fan-in init N(0, 1/d_in) (see module doc)
    qk_gain: float = 1.0     # extra scale of the q/k rows (1 = plain fan-in init)
    judge: bool = False      # install the judge circuit (base models)
    cue_gain: float = 4.0
    digit_gain: float = 6.0
    digit_noise: float = 1.0
    judge_offsets: tuple = ()  # per-digit gain offsets (tools/calibrate_judge.py)
    embed_std: float = 0.0   # embedding init std (0 -> 0.02)
    succ_gain: float = 0.0   # successor circuit (module doc); 0 = off
    probe_gain: float = 0.0  # judge probe head output scale (module doc); 0 = off
    probe_scale: float = 6.0  # per-RoPE-pair amplitude of the probe head's q / k
    probe_offset: int = 36   # cue-to-probed-token distance (last candidate word)
    # tensor parallelism (tp_spec): this rank's shard of a model split `tp_world` ways
    tp_world: int = 1
    tp_rank: int = 0
    embed_rows: int = 0      # embedding rows when they differ from the LM-head shard (0: same)
    vocab_base: int = 0      # global id of this rank's LM-head row 0

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def qkv_rows(self) -> int:
        return self.q_dim + 2 * self.kv_dim

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    def body_params(self) -> int:
        d = self.d_model
        per_layer = (self.qkv_rows * d + self.qkv_rows + self.q_dim * d
                     + 3 * self.d_ffn * d + 2 * d)
        return self.n_layers * per_layer + d

    def head_params(self) -> int:
        return self.vocab_rows * self.d_model

    def kv_bytes_per_token(self) -> int:
        return self.n_layers * 2 * self.kv_dim * 2

    def decode_bytes(self, ctx: int) -> int:
        """Algorithmic HBM bytes of one decode token at context ``ctx``
        (SURVEY.md §8d): all weights once plus the KV of ctx+1 positions.
        The embedding row is one row, not the table."""
        return 2 * (self.body_params() + self.head_params()) + (ctx + 1) * self.kv_bytes_per_token()


    def prefill_cost(self, start: int, n: int, head_rows: int = 1,
                     chunk: int = 256) -> tuple[float, float]:
        """Algorithmic (HBM bytes, flops) of prefilling ``n`` rows at
        positions ``start``.. in chunks of ``chunk`` rows (SURVEY §8d verify
        row): per chunk the body weights once, the K/V of the context read
        once and the new rows' K/V written; 2*M*P_body GEMM flops plus the
        causal attention 4*L*H*128*M*(ctx + M/2); the LM head once for
        ``head_rows`` readout rows."""
        by = fl = 0.0
        kvb = self.kv_bytes_per_token()
        attn = 4 * self.n_layers * self.n_heads * self.head_dim
        c0 = 0
        while c0 < n:
            m = min(chunk, n - c0)
            s = start + c0
            by += 2 * self.body_params() + (s + m) * kvb + m * kvb
            fl += 2 * m * self.body_params() + attn * m * (s + m / 2)
            c0 += m
        if head_rows:
            by += 2 * self.head_params()
            fl += 2 * head_rows * self.head_params()
        return by, fl


V_QWEN_DRAFT = 151_936
V_QWEN_BASE = 152_064

MODELS: dict[str, ModelSpec] = {
    # C1 tiny pair (SURVEY.md §8 "C1 (proposed)"; head_dim kept at 128 so the
    # tiny pair runs the exact kernels of the full-size models)
    "tiny-draft": ModelSpec("tiny-draft", 2, 128, 2, 1, 512, 4096, 4096, rope_theta=10_000.0),
    "tiny-base": ModelSpec("tiny-base", 4, 256, 4, 2, 1024, 4160, 4096, judge=True,
                           judge_offsets=(-0.5, -0.125, -0.5, 0.375, 0.5, 0.25, 0.0, 0.375, 0.25, -0.5)),
    # public model-card shapes; embed_std / succ_gain: the successor circuit
    # (module doc); judge offsets measured on the B200 by
    # tools/calibrate_judge.py --gpu (seed 0)
    "r1-1.5b": ModelSpec("r1-1.5b", 28, 1536, 12, 2, 8960, V_QWEN_DRAFT, V_QWEN_DRAFT,
                         rope_theta=10_000.0, embed_std=1.0, succ_gain=0.8),
    "qwen2.5-7b": ModelSpec("qwen2.5-7b", 28, 3584, 28, 4, 18944, V_QWEN_BASE, V_QWEN_DRAFT,
                            judge=True, embed_std=1.0, succ_gain=0.8, cue_gain=6.0,
                            digit_gain=12.0, digit_noise=2.0, probe_gain=30.0,
                            judge_offsets=(-1.0, 2.125, -0.5, -2.0, -1.625, 1.25, -0.25, 0.125,
                                           0.0, 2.125)),
    "qwq-32b": ModelSpec("qwq-32b", 64, 5120, 40, 8, 27648, V_QWEN_BASE, V_QWEN_DRAFT,
                         judge=True, embed_std=1.0, succ_gain=0.8, cue_gain=6.0,
                         digit_gain=12.0, digit_noise=2.0, probe_gain=30.0,
                         judge_offsets=(-2.5, 0.25, 3.75, -1.25, 3.5, -0.75, -2.625, -2.75, 0.875,
                                        1.125)),
}

PAIRS = {
    "tiny": ("tiny-draft", "tiny-base"),
    "1.5b+7b": ("r1-1.5b", "qwen2.5-7b"),
    "1.5b+32b": ("r1-1.5b", "qwq-32b"),
}


def tp_spec(spec: ModelSpec, rank: int, world: int) -> ModelSpec:
    """Rank `rank`'s shard of `spec` under Megatron-style tensor parallelism
    (SURVEY §8e): q/k/v heads and gate/up units column-parallel, O and down
    row-parallel (their partial outputs all-reduced), LM head vocab-parallel,
    embedding and norms replicated."""
    if world == 1:
        return spec
    if spec.n_heads % world or spec.n_kv_heads % world:
        raise ValueError(f"{spec.name}: heads {spec.n_heads}/{spec.n_kv_heads} not divisible by {world}")
    if spec.d_ffn % (GU_BLOCK * world):
        raise ValueError(f"{spec.name}: d_ffn {spec.d_ffn} not divisible by {GU_BLOCK * world}")
    if spec.vocab_rows % (32 * world):
        raise ValueError(f"{spec.name}: vocab rows {spec.vocab_rows} not divisible by {32 * world}")
    vr = spec.vocab_rows // world
    base = rank * vr
    return replace(spec, name=f"{spec.name}-tp{rank}of{world}", n_heads=spec.n_heads // world,
                   n_kv_heads=spec.n_kv_heads // world, d_ffn=spec.d_ffn // world,
                   vocab_rows=vr, vocab_text=max(0, min(vr, spec.vocab_text - base)),
                   embed_rows=spec.vocab_rows, vocab_base=base, tp_world=world, tp_rank=rank)


def shard_tensor(name: str, t: torch.Tensor, spec: ModelSpec, rank: int, world: int) -> torch.Tensor:
    """Rank `rank`'s slice of the full parameter `name` (see tp_spec)."""
    if world == 1:
        return t
    leaf = name.rsplit(".", 1)[-1]
    H, KV, f, hd = spec.n_heads // world, spec.n_kv_heads // world, spec.d_ffn // world, spec.head_dim
    qd, kd = spec.q_dim, spec.kv_dim
    q_rows = slice(rank * H * hd, (rank + 1) * H * hd)
    if leaf in ("wqkv", "bqkv"):
        k_rows = slice(qd + rank * KV * hd, qd + (rank + 1) * KV * hd)
        v_rows = slice(qd + kd + rank * KV * hd, qd + kd + (rank + 1) * KV * hd)
        return torch.cat([t[q_rows], t[k_rows], t[v_rows]]).contiguous()
    if leaf == "wo":
        return t[:, q_rows].contiguous()
    if leaf == "wgu":                                     # whole 32-row gate/up blocks
        return t[2 * rank * f:2 * (rank + 1) * f].contiguous()
    if leaf == "wd":
        return t[:, rank * f:(rank + 1) * f].contiguous()
    if leaf == "lm_head":
        vr = spec.vocab_rows // world
        return t[rank * vr:(rank + 1) * vr].contiguous()
    return t                                              # embed, norms: replicated


def shard_weights(full: dict[str, torch.Tensor], spec: ModelSpec, rank: int,
                  world: int) -> dict[str, torch.Tensor]:
    """Slice a full model's weights into rank `rank`'s shard (see tp_spec)."""
    return {k: shard_tensor(k, v, spec, rank, world) for k, v in full.items()}


def make_tp_weights(spec: ModelSpec, rank: int, world: int, seed: int = 0,
                    device: str = "cpu") -> dict[str, torch.Tensor]:
    """Rank `rank`'s shard, generated tensor by tensor (peak memory: one full
    tensor), identical to slicing make_weights(spec)."""
    return {name: shard_tensor(name, make_tensor(spec, seed, name, device), spec, rank, world)
            for name in tensor_shapes(spec)}


def get_spec(name: str, **overrides) -> ModelSpec:
    spec = MODELS[name]
    return replace(spec, **overrides) if overrides else spec


# --------------------------------------------------------------------------
# weights
# --------------------------------------------------------------------------

def tensor_shapes(spec: ModelSpec) -> dict[str, tuple[int, ...]]:
    """Name -> shape for every parameter (row-major, out_features first).

    ``wqkv`` stacks q, k, v rows; ``wgu`` interleaves gate and up rows in
    blocks of 16 (rows 32b..32b+15 gate, 32b+16..32b+31 up), the layout the
    fused gate/up kernels consume.
    """
    d = spec.d_model
    shapes: dict[str, tuple[int, ...]] = {"embed": (spec.embed_rows or spec.vocab_rows, d), "ln_f": (d,),
                                          "lm_head": (spec.vocab_rows, d)}
    for i in range(spec.n_layers):
        p = f"layers.{i}."
        shapes[p + "ln1"] = (d,)
        shapes[p + "wqkv"] = (spec.qkv_rows, d)
        shapes[p + "bqkv"] = (spec.qkv_rows,)
        shapes[p + "wo"] = (d, spec.q_dim)
        shapes[p + "ln2"] = (d,)
        shapes[p + "wgu"] = (2 * spec.d_ffn, d)
        shapes[p + "wd"] = (d, spec.d_ffn)
    return shapes


GU_BLOCK = 16


def gu_interleave(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    f, d = gate.shape
    return torch.stack([gate.view(f // GU_BLOCK, GU_BLOCK, d),
                        up.view(f // GU_BLOCK, GU_BLOCK, d)], dim=1).reshape(2 * f, d)


def gu_split(wgu: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    two_f, d = wgu.shape
    v = wgu.view(two_f // (2 * GU_BLOCK), 2, GU_BLOCK, d)
    return v[:, 0].reshape(-1, d), v[:, 1].reshape(-1, d)


def _seed_for(spec: ModelSpec, seed: int, name: str) -> int:
    return derive_seed("weights", spec.name, seed, name) & ((1 << 63) - 1)


def _judge_direction(spec: ModelSpec, seed: int) -> torch.Tensor:
    g = torch.Generator().manual_seed(_seed_for(spec, seed, "judge.u"))
    u = torch.randn(spec.d_model, generator=g, dtype=torch.float64)
    return (u / u.norm()).to(torch.float32)


def init_std(spec: ModelSpec, name: str) -> float:
    if spec.init_std > 0:
        return spec.init_std
    leaf = name.rsplit(".", 1)[-1]
    if leaf == "embed" and spec.embed_std > 0:
        return spec.embed_std
    if leaf in ("bqkv", "embed"):
        return 0.02
    fan_in = {"wo": spec.q_dim, "wd": spec.d_ffn}.get(leaf, spec.d_model)
    return 1.0 / math.sqrt(fan_in)


def make_tensor(spec: ModelSpec, seed: int, name: str, device: str = "cpu") -> torch.Tensor:
    """Generate one parameter as bf16 on ``device`` (deterministic per device
    type: the CPU generator for parity slices, the CUDA one for full models)."""
    shape = tensor_shapes(spec)[name]
    leaf = name.rsplit(".", 1)[-1]
    if leaf in ("ln1", "ln2", "ln_f"):
        return torch.ones(shape, dtype=torch.bfloat16, device=device)
    g = torch.Generator(device=device).manual_seed(_seed_for(spec, seed, name))
    t = torch.randn(shape, generator=g, dtype=torch.float32, device=device)
    t.mul_(init_std(spec, name))
    if leaf == "wqkv":
        t[: spec.q_dim + spec.kv_dim].mul_(spec.qk_gain)
    if spec.judge and name == "embed":
        u = _judge_direction(spec, seed).to(device)
        t[JUDGE_CUE_ID] = spec.cue_gain * math.sqrt(spec.d_model) * u
    if spec.judge and name == "lm_head":
        u = _judge_direction(spec, seed).to(device)
        offs = spec.judge_offsets or (0.0,) * len(DIGIT_IDS)
        for dgt in DIGIT_IDS:
            r = t[dgt] * spec.digit_noise
            r = r - (r @ u) * u
            t[dgt] = r + ((spec.digit_gain + offs[dgt]) / math.sqrt(spec.d_model)) * u
        if spec.vocab_rows > spec.vocab_text:
            t[spec.vocab_text] = u / math.sqrt(spec.d_model)  # cue-alignment probe
    if spec.judge and spec.probe_gain > 0 and name.startswith(f"layers.{spec.n_layers - 1}."):
        _install_probe(spec, seed, leaf, t)
    if spec.succ_gain > 0 and name == "lm_head":
        # successor circuit: row v reads the (unit) embedding of v's predecessor
        emb = make_tensor(spec, seed, "embed", device).float()
        lo, hi = successor_range(spec.vocab_text)
        pred = successor_perm(spec.vocab_text, seed)[1].to(device)
        rows = torch.arange(lo, hi, device=device)
        src = emb[pred[rows]]
        t[rows] += spec.succ_gain * (src / src.norm(dim=1, keepdim=True))
        del emb, src
    return t.to(torch.bfloat16)


def probe_pairs(spec: ModelSpec) -> np.ndarray:
    """RoPE pairs the probe head uses: frequencies in [0.02, 1] rad/token,
    enough to resolve single positions without aliasing over 16K tokens."""
    half = spec.head_dim // 2
    inv = spec.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / spec.head_dim)
    return np.where((inv >= 0.02) & (inv <= 1.0))[0]


def _install_probe(spec: ModelSpec, seed: int, leaf: str, t: torch.Tensor) -> None:
    """Judge probe head (last layer, q head 0 / kv head 0; module doc)."""
    hd, half, dev = spec.head_dim, spec.head_dim // 2, t.device
    P = probe_pairs(spec)
    inv = spec.rope_theta ** (-P.astype(np.float64) * 2.0 / spec.head_dim)
    c = spec.probe_scale
    if leaf == "wqkv":
        u = _judge_direction(spec, seed).to(dev)
        qv = torch.zeros(hd, device=dev)
        qv[torch.as_tensor(P, device=dev)] = c
        t[:hd] = torch.outer(qv, u) / math.sqrt(spec.d_model)
        t[spec.q_dim: spec.q_dim + hd] = 0.0
    elif leaf == "bqkv":
        t[:hd] = 0.0
        kv = torch.zeros(hd, dtype=torch.float64)
        kv[torch.as_tensor(P)] = c * torch.from_numpy(np.cos(inv * spec.probe_offset))
        kv[torch.as_tensor(P + half)] = c * torch.from_numpy(np.sin(inv * spec.probe_offset))
        t[spec.q_dim: spec.q_dim + hd] = kv.to(dev, torch.float32)
    elif leaf == "wo":
        t[:, :hd] *= spec.probe_gain


def successor_range(n_text: int) -> tuple[int, int]:
    """Ids the successor circuit permutes: the ordinary words (``vocab``)."""
    from .vocab import FIRST_WORD_ID

    return FIRST_WORD_ID, n_text


def successor_perm(n_text: int, seed: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
    """(succ, pred): a seeded random permutation of the ordinary word ids
    and its inverse, as int64 tables over [0, n_text) (identity outside the
    ordinary range).  Keyed by the vocabulary, not the model, so a draft and
    a base sharing a vocabulary share their preferred successors."""
    lo, hi = successor_range(n_text)
    g = torch.Generator().manual_seed(derive_seed("successor", n_text, seed) & ((1 << 63) - 1))
    perm = torch.randperm(hi - lo, generator=g) + lo
    succ = torch.arange(n_text, dtype=torch.int64)
    succ[lo:hi] = perm
    pred = torch.arange(n_text, dtype=torch.int64)
    pred[perm] = torch.arange(lo, hi, dtype=torch.int64)
    return succ, pred


def make_weights(spec: ModelSpec, seed: int = 0, device: str = "cpu",
                 layers: list[int] | None = None) -> dict[str, torch.Tensor]:
    """All (or a layer subset of) parameters as bf16 tensors on ``device``."""
    out = {}
    for name in tensor_shapes(spec):
        if layers is not None and name.startswith("layers."):
            if int(name.split(".")[1]) not in layers:
                continue
        out[name] = make_tensor(spec, seed, name, device)
    return out


def rope_table(spec: ModelSpec, max_pos: int) -> torch.Tensor:
    """fp32 [max_pos, head_dim/2, 2] (cos, sin) computed in float64 once, so
    the kernels and the CPU oracle rotate by bit-identical factors."""
    half = spec.head_dim // 2
    inv = spec.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / spec.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    tab = np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)
    return torch.from_numpy(tab)


# --------------------------------------------------------------------------
# judge calibration (see module doc)
# --------------------------------------------------------------------------

def judge_calibration_prompts(spec: ModelSpec, n: int = 24, cot_step: int = 25,
                              chain: bool = False, one_chain: bool = False) -> list[list[int]]:
    """Token ids of ``n`` synthetic verify prompts (64-word problem, a CoT of
    0, cot_step, .. words, a 24-word candidate), seeded and model-independent.
    ``chain``: the CoT and candidate follow the successor circuit's
    permutation from a random start word -- the text the successor-circuit
    models actually generate, so the calibration sees loop-like contexts."""
    from .domain import render_verification_prompt
    from .vocab import shared_vocab

    vocab = shared_vocab(spec.vocab_text)
    lo, hi = vocab.ordinary_range()
    rng = np.random.default_rng(20250410)
    succ = successor_perm(vocab.n_text)[0].tolist() if chain else None
    out = []
    base_ids = [int(x) for x in rng.integers(lo, hi, size=64 + cot_step * n + 24)]
    for i in range(n):
        c = cot_step * i
        ids = (base_ids[:64 + c + 24] if one_chain
               else [int(x) for x in rng.integers(lo, hi, size=64 + c + 24)])
        if chain:
            for k in range(65, len(ids)):
                ids[k] = succ[ids[k - 1]]
        w = [vocab.words[x] for x in ids]
        prompt = render_verification_prompt(" ".join(w[:64]), " ".join(w[64:64 + c]) + " ",
                                            " ".join(w[64 + c:]) + " ")
        out.append(vocab.encode(prompt))
    return out


def judge_offsets_update(spec: ModelSpec, last_logits: list[torch.Tensor]) -> tuple:
    """One calibration step: new per-digit gain offsets that equalise the
    digits' mean logit at the cue, from the last-position logits of the
    calibration prompts (probe row = cue alignment)."""
    L = torch.stack([x.float().cpu() for x in last_logits])
    mu = L[:, list(DIGIT_IDS)].mean(0)
    probe = float(L[:, spec.vocab_text].mean())
    delta = -(mu - mu.mean()) / probe
    old = spec.judge_offsets or (0.0,) * len(DIGIT_IDS)
    return tuple(round((o + float(d)) * 8) / 8 for o, d in zip(old, delta))
