"""Layer-streamed fp32 oracle over a prefix tree of sequences -- TEST
INFRASTRUCTURE ONLY (see ``ref_model.py`` for what the oracle restates and
why the model arithmetic has no reference source).

Why a second form of the oracle
-------------------------------
``RefModel`` keeps the whole model resident and runs one sequence at a time
with a KV cache: fine for the tiny pair, too slow and too large for a full
32B-shape trajectory (64 layers, 8K-token contexts, hundreds of backend
calls).  ``TreeOracle`` computes *the same function* (identical operation
order and bf16 storage points as ``RefModel.forward``) for every sequence a
trajectory's backend calls fed to the model, with two changes of schedule
only:

* **prefix tree**: every call's fed sequence (generation prompt + generated
  tokens, verification prompt) is inserted into a compressed trie, so shared
  prefixes -- the CoT every call repeats -- are computed once.  A position
  attends to exactly the positions of its own sequence before it (ancestor
  nodes in the trie, earlier positions of its node): the semantics of the
  reference's prefix-cache streams (``_PrefixLedger``, ``engine.py:161-186``)
  without any cache state;
* **layer streaming**: the outer loop is over layers; each layer's bf16
  weights are fetched (``fetch(name)``), upcast to the oracle dtype, applied
  to every trie position, and dropped.  Peak memory is one layer plus the
  activations, so the 32B shape runs in fp32 (and fp64, for the noise floor)
  where the whole model would need 131 / 262 GB.

The arithmetic runs with torch on ``device``: on the CPU for small shapes and
the CPU cross-check, on the GPU for full-depth 7B/32B trajectories (fp32
without TF32, fp64).  ``tests/test_tree_oracle.py`` pins TreeOracle to
``RefModel`` on the CPU, and the device execution to the CPU one.

Only summaries of each wanted position's logits leave the oracle (argmax,
top-2 margin, the logit gap to a given token, the judge readout and its
ambiguity), so 152K-wide logits are never stored for thousands of rows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Sequence

import torch

from paper_2504_07891_b200.shapes import ModelSpec, gu_split, rope_table


def _r(x: torch.Tensor, on: bool) -> torch.Tensor:
    return x.to(torch.bfloat16).to(x.dtype) if on else x


def _lcp(a: Sequence[int], b: Sequence[int]) -> int:
    n = min(len(a), len(b))
    if list(a[:n]) == list(b[:n]):
        return n
    lo, hi = 0, n
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if list(a[lo:mid]) == list(b[lo:mid]):
            lo = mid
        else:
            hi = mid
    return lo


@dataclass
class _Node:
    tokens: list
    parent: "_Node | None"
    start: int
    children: dict = field(default_factory=dict)
    slot0: int = 0
    dfs_in: int = 0
    dfs_out: int = 0


class PrefixTrie:
    """Compressed trie of token sequences; slots laid out in DFS preorder so
    every ancestor position has a smaller slot than its descendants."""

    def __init__(self) -> None:
        self.root = _Node([], None, 0)
        self.seqs: list[list[int]] = []

    def insert(self, seq: Sequence[int]) -> int:
        seq = list(seq)
        self.seqs.append(seq)
        node, i = self.root, 0
        while i < len(seq):
            child = node.children.get(seq[i])
            if child is None:
                node.children[seq[i]] = _Node(seq[i:], node, i)
                break
            j = _lcp(child.tokens, seq[i:i + len(child.tokens)])
            if j < len(child.tokens):  # split child at j
                tail = _Node(child.tokens[j:], child, child.start + j, child.children)
                for c in tail.children.values():
                    c.parent = tail
                child.tokens = child.tokens[:j]
                child.children = {tail.tokens[0]: tail}
            i += j
            node = child
        return len(self.seqs) - 1

    def finalize(self) -> None:
        self.nodes: list[_Node] = []
        slot, clock = 0, 0
        stack = [(self.root, False)]
        while stack:
            n, done = stack.pop()
            if done:
                n.dfs_out = clock
                clock += 1
                continue
            n.dfs_in = clock
            clock += 1
            n.slot0 = slot
            slot += len(n.tokens)
            self.nodes.append(n)
            stack.append((n, True))
            for c in sorted(n.children.values(), key=lambda c: c.tokens[0], reverse=True):
                stack.append((c, False))
        self.n_slots = slot

    def slot_of(self, seq_index: int, pos: int) -> int:
        return self.slots_of(seq_index, [pos])[0]

    def slots_of(self, seq_index: int, positions: Sequence[int]) -> list[int]:
        """Slots of positions of sequence ``seq_index`` (after finalize)."""
        import bisect

        seq = self.seqs[seq_index]
        path, node, i = [], self.root, 0
        while i < len(seq):
            node = node.children[seq[i]]
            path.append(node)
            i += len(node.tokens)
        starts = [n.start for n in path]
        out = []
        for p in positions:
            n = path[bisect.bisect_right(starts, p) - 1]
            out.append(n.slot0 + p - n.start)
        return out

    def slot_tables(self) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
        """Per slot: token id, position, dfs_in, dfs_out of its node."""
        ids, pos, din, dout = [], [], [], []
        for n in self.nodes:
            k = len(n.tokens)
            ids.extend(n.tokens)
            pos.extend(range(n.start, n.start + k))
            din.extend([n.dfs_in] * k)
            dout.extend([n.dfs_out] * k)
        T = lambda x: torch.tensor(x, dtype=torch.long)  # noqa: E731
        return T(ids), T(pos), T(din), T(dout)


class TreeOracle:
    """fp32 (or fp64) forward of every position of a ``PrefixTrie``.

    ``fetch(name) -> tensor`` returns a parameter as stored (bf16, any
    device); names follow ``shapes.tensor_shapes``."""

    def __init__(self, spec: ModelSpec, fetch: Callable[[str], torch.Tensor], *,
                 device: str | torch.device = "cpu", dtype: torch.dtype = torch.float32,
                 exact_fp32: bool = False, attn_bytes: float = 2e9, mlp_rows: int = 4096) -> None:
        self.spec = spec
        self.fetch = fetch
        self.device = torch.device(device)
        self.dtype = dtype
        self.round = not exact_fp32
        self.attn_bytes = attn_bytes
        self.mlp_rows = mlp_rows

    def _w(self, name: str) -> torch.Tensor:
        return self.fetch(name).to(self.device).to(self.dtype).contiguous()

    def _norm(self, h: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        ms = (h * h).mean(dim=-1, keepdim=True)
        return _r(h * torch.rsqrt(ms + self.spec.rms_eps) * w, self.round)

    @torch.no_grad()
    def hidden(self, trie: PrefixTrie) -> torch.Tensor:
        """Final-norm hidden state [n_slots, d] of every trie position."""
        spec, rd, dev, dt = self.spec, self.round, self.device, self.dtype
        if self.device.type == "cuda":
            torch.backends.cuda.matmul.allow_tf32 = False
        trie.finalize()
        ids, pos, din, dout = (t.to(dev) for t in trie.slot_tables())
        S = ids.numel()
        hd, H, KV, G = spec.head_dim, spec.n_heads, spec.n_kv_heads, spec.group
        scale = 1.0 / math.sqrt(hd)
        tab = rope_table(spec, int(pos.max()) + 1).to(dev).to(dt)
        cos, sin = tab[..., 0][pos][:, None, :], tab[..., 1][pos][:, None, :]

        def rope(x):
            half = x.shape[-1] // 2
            x1, x2 = x[..., :half], x[..., half:]
            return torch.cat([x1 * cos[: x.shape[0]] - x2 * sin[: x.shape[0]],
                              x2 * cos[: x.shape[0]] + x1 * sin[: x.shape[0]]], dim=-1)

        h = self.fetch("embed").to(dev)[ids].to(dt)
        elem = torch.finfo(dt).bits // 8
        for li in range(spec.n_layers):
            p = f"layers.{li}."
            wqkv, bqkv, wo = self._w(p + "wqkv"), self._w(p + "bqkv"), self._w(p + "wo")
            x = self._norm(h, self._w(p + "ln1"))
            qkv = x @ wqkv.T + bqkv
            del x
            q = _r(rope(qkv[:, : spec.q_dim].view(S, H, hd)), rd)
            k = _r(rope(qkv[:, spec.q_dim: spec.q_dim + spec.kv_dim].view(S, KV, hd)), rd)
            v = _r(qkv[:, spec.q_dim + spec.kv_dim:].view(S, KV, hd), rd)
            del qkv
            o = torch.empty(S, spec.q_dim, device=dev, dtype=dt)
            a = 0
            while a < S:
                # keys of slots [0, b): ancestors precede descendants in DFS order
                # score + probability tensors [H, rows, b] within attn_bytes
                rows = max(16, int(self.attn_bytes / (min(S, a + 1024) * H * elem * 3)))
                b = min(S, a + rows)
                Kx = k[:b].repeat_interleave(G, dim=1).permute(1, 2, 0)     # [H, hd, b]
                Vx = v[:b].repeat_interleave(G, dim=1).permute(1, 0, 2)     # [H, b, hd]
                s = torch.bmm(q[a:b].permute(1, 0, 2), Kx) * scale            # [H, n, b]
                vis = ((din[None, :b] <= din[a:b, None]) & (dout[a:b, None] <= dout[None, :b])
                       & (pos[None, :b] <= pos[a:b, None]))
                s = s.masked_fill(~vis[None], float("-inf"))
                pr = torch.softmax(s, dim=-1)
                o[a:b] = torch.bmm(pr, Vx).permute(1, 0, 2).reshape(b - a, spec.q_dim)
                del Kx, Vx, s, vis, pr
                a = b
            o = _r(o, rd)
            h = h + o @ wo.T
            del o, q, k, v, wqkv, bqkv, wo
            gate, up = gu_split(self.fetch(p + "wgu"))
            wg = gate.to(dev).to(dt).contiguous()
            wu = up.to(dev).to(dt).contiguous()
            wd = self._w(p + "wd")
            ln2 = self._w(p + "ln2")
            for r0 in range(0, S, self.mlp_rows):
                r1 = min(S, r0 + self.mlp_rows)
                x2 = self._norm(h[r0:r1], ln2)
                g = x2 @ wg.T
                u = x2 @ wu.T
                act = _r(torch.nn.functional.silu(g) * u, rd)
                h[r0:r1] = h[r0:r1] + act @ wd.T
                del x2, g, u, act
            del wg, wu, wd, gate, up
        return self._norm(h, self._w("ln_f"))

    @torch.no_grad()
    def logits_rows(self, hidden: torch.Tensor, slots: Sequence[int], chunk: int = 256):
        """Yield (slot indices, fp32/fp64 logits [n, V]) for ``slots`` in chunks."""
        head = self._w("lm_head")
        for c0 in range(0, len(slots), chunk):
            sl = list(slots[c0:c0 + chunk])
            idx = torch.tensor(sl, dtype=torch.long, device=hidden.device)
            yield sl, hidden[idx] @ head.T


# --------------------------------------------------------------------------
# summaries (what the parity tests compare)
# --------------------------------------------------------------------------

def choice_summary(row: torch.Tensor, n_text: int, choice: int | None) -> dict:
    """Greedy argmax (first index on ties), top1 - top2 margin, and the gap
    top1 - logit[choice] of a device's choice (0 when it is the argmax)."""
    r = row[:n_text]
    top = torch.topk(r, 2)
    arg = int(torch.argmax(r))
    out = {"argmax": arg, "margin": float(top.values[0] - top.values[1])}
    if choice is not None:
        out["gap"] = float(r[arg] - r[choice]) if 0 <= choice < n_text else float("inf")
    return out


def readout_ambiguity(row: torch.Tensor, n_text: int, digit_ids=tuple(range(10))) -> float:
    """Smallest logit gap that decides the judge readout (``extract_score``
    over the top-10 of the position, ``base.py:106-126``): between the best
    two member digits, between any digit and the top-10 boundary, and -- when
    no digit is a member -- between the argmax and the runner-up (the sampled
    token's first digit decides).  A readout whose gap is below the logit
    tolerance can legitimately differ between two fp32 implementations."""
    r = row[:n_text].double()
    top = torch.topk(r, 11).values
    v9, v10 = float(top[9]), float(top[10])
    d = r[list(digit_ids)]
    gaps = [abs(float(x) - v9) for x in d] + [abs(float(x) - v10) for x in d]
    members = sorted((float(x) for x in d if float(x) >= v9), reverse=True)
    if len(members) >= 2:
        gaps.append(members[0] - members[1])
    if not members:
        gaps.append(float(top[0] - top[1]))
    return min(gaps)
