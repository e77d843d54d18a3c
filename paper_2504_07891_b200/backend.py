"""``B200Backend``: the reference ``Backend`` plugin API on sm_100a kernels.

PyTorch only owns memory here: weights, the K/V page pools, the workspace and
small staging buffers are torch CUDA tensors whose raw pointers cross the
C-ABI (``native.py``).  All arithmetic -- prefill, greedy decode with the
device-side stop test, the judge readout and threshold compare -- runs in the
native library; per call the host uploads the fresh token ids (4 B each) and
reads back the generated ids (``sr_generate``) or a 16-byte readout
(``sr_score``).

Pages: each prefix-cache stream (``host.Stream``) owns a list of page ids and
a device page table.  Rolling a stream back to its common prefix frees the
pages past it; a prefill commits new positions into freshly allocated pages.
When the pool runs dry the least recently used other stream is evicted.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import ctypes as C
import torch

from . import native
from .domain import BackendProfile, BackendRole
from .host import ModelBackend, Readout, Stream
from .shapes import (PAIRS, ModelSpec, get_spec, make_tp_weights, make_weights, rope_table,
                     shard_weights, tensor_shapes, tp_spec)
from .vocab import CLASS_END_THINK, CLASS_STOP, Vocab, shared_vocab

PAGE = native.SR_PAGE


def first_digit_table(vocab: Vocab, n_rows: int) -> torch.Tensor:
    """int8 [n_rows]: first '0'-'9' character of each token's text, or -1."""
    out = torch.full((n_rows,), -1, dtype=torch.int8)
    for i in range(vocab.n_text):
        for ch in vocab.render_one(i):
            if "0" <= ch <= "9":
                out[i] = ord(ch) - 48
                break
    return out


def decode_tiles(w: torch.Tensor) -> torch.Tensor:
    """A [N][K] bf16 matrix in the persistent decode kernel's tile-major
    layout (``sr_model_set_decode_tiles``): 32-row x tc-column tiles
    (tc = min(K, 256)) in (row block, k tile) order, each as tc/64 boxes of
    [32][64] with the 128-B swizzle applied -- the 16-B chunk j of row r
    stored at chunk position j ^ (r & 7) -- so a tile is one contiguous 16 KB
    bulk copy whose shared-memory image ``ldmatrix`` reads conflict free."""
    N, K = w.shape
    tc = min(K, 256)
    if N % 32 or K % tc or tc % 64:
        raise ValueError(f"decode tiles need N % 32 == 0 and K % {tc} == 0 (got {N} x {K})")
    x = w.view(N // 32, 32, K // tc, tc // 64, 8, 8).permute(0, 2, 3, 1, 4, 5)
    r = torch.arange(32, device=w.device)[:, None].expand(32, 8)
    src = torch.arange(8, device=w.device)[None, :] ^ (r & 7)  # chunk stored at position p
    return x[:, :, :, r, src, :].contiguous().view(-1)


class DeviceModel:
    """One model's weights, K/V page pools, workspace and native handle."""

    def __init__(self, spec: ModelSpec, weights: dict[str, torch.Tensor], *, max_pos: int,
                 n_pages: int, max_tokens: int = 256, max_new: int = 256,
                 device: str | torch.device = "cuda", decode_layout: bool = True) -> None:
        self.lib = native.load()
        self.spec = spec
        self.device = torch.device(device)
        self.max_pos = max_pos
        self.max_new = max_new
        self.n_pages = n_pages
        self.weights = {k: v.to(self.device, torch.bfloat16).contiguous() for k, v in weights.items()}
        for name, shape in tensor_shapes(spec).items():
            if tuple(self.weights[name].shape) != shape:
                raise ValueError(f"weight {name} has shape {tuple(self.weights[name].shape)}")
        self.rope = rope_table(spec, max_pos).to(self.device).contiguous()
        pool_elems = spec.n_layers * n_pages * spec.n_kv_heads * PAGE * spec.head_dim
        self.k_pool = torch.zeros(pool_elems, dtype=torch.bfloat16, device=self.device)
        self.v_pool = torch.zeros(pool_elems, dtype=torch.bfloat16, device=self.device)
        self.desc = native.ModelDesc(
            n_layers=spec.n_layers, d_model=spec.d_model, n_heads=spec.n_heads,
            n_kv_heads=spec.n_kv_heads, head_dim=spec.head_dim, d_ffn=spec.d_ffn,
            vocab_rows=spec.vocab_rows, vocab_text=spec.vocab_text, rms_eps=spec.rms_eps,
            max_pos=max_pos, max_tokens=max_tokens, max_new=max_new, n_pages=n_pages,
            tp_world=spec.tp_world, tp_rank=spec.tp_rank, vocab_base=spec.vocab_base)
        ws = self.lib.sr_workspace_bytes(C.byref(self.desc))
        if ws == 0:
            raise native.NativeError("sr_workspace_bytes", -1, self.lib.sr_last_error().decode())
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        W = self.weights
        self._layer_arr = (native.LayerPtrs * spec.n_layers)()
        for i in range(spec.n_layers):
            p = f"layers.{i}."
            self._layer_arr[i] = native.LayerPtrs(*(W[p + n].data_ptr() for n in (
                "ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wd")))
        ptrs = native.ModelPtrs(
            embed=W["embed"].data_ptr(), ln_f=W["ln_f"].data_ptr(),
            lm_head=W["lm_head"].data_ptr(), layers=self._layer_arr,
            rope=self.rope.data_ptr(), k_pool=self.k_pool.data_ptr(),
            v_pool=self.v_pool.data_ptr(), workspace=self.workspace.data_ptr())
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream().cuda_stream
            native.check("sr_model_create", self.lib.sr_model_create(
                C.byref(self.desc), C.byref(ptrs), C.c_void_p(stream), C.byref(handle)))
        self.handle = handle
        # decode-layout copy of the streamed matrices (the row-major weights
        # stay for prefill): one contiguous bulk copy per 16 KB tile, GEMVs on
        # the tensor cores (K3)
        self.tiles: list[torch.Tensor] = []
        if decode_layout:
            names = [f"layers.{i}.{n}" for i in range(spec.n_layers) for n in ("wqkv", "wo", "wgu", "wd")]
            self.tiles = [decode_tiles(W[n]) for n in names + ["lm_head"]]
            arr = (C.c_uint64 * len(self.tiles))(*(t.data_ptr() for t in self.tiles))
            native.check("sr_model_set_decode_tiles", self.lib.sr_model_set_decode_tiles(handle, arr))
        self.free_pages = list(range(n_pages - 1, -1, -1))
        self.max_tokens = max_tokens
        # staging
        self.ids_host = torch.empty(max_pos, dtype=torch.int32, pin_memory=True)
        self.ids_dev = torch.empty(max_pos, dtype=torch.int32, device=self.device)
        self.out_dev = torch.zeros(2 + max_new, dtype=torch.int32, device=self.device)
        self.margin_dev = torch.zeros(max_new, dtype=torch.float32, device=self.device)
        self.out_host = torch.empty(2 + max_new, dtype=torch.int32, pin_memory=True)
        self.margin_host = torch.empty(max_new, dtype=torch.float32, pin_memory=True)
        # multi-sequence passes: (position, page) per row, outputs per sequence
        self.meta_host = torch.empty(2 * max_tokens, dtype=torch.int32, pin_memory=True)
        self.meta_dev = torch.empty(2 * max_tokens, dtype=torch.int32, device=self.device)
        self.batch_out = torch.zeros(4 * 64, dtype=torch.int32, device=self.device)
        self.batch_margins = torch.zeros(64, dtype=torch.float32, device=self.device)
        self.readout_dev = torch.zeros(4, dtype=torch.int32, device=self.device)
        self.readout_host = torch.empty(4, dtype=torch.int32, pin_memory=True)

    def __del__(self) -> None:
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.sr_model_destroy(h)
            except Exception:
                pass

    @property
    def stream_ptr(self) -> C.c_void_p:
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def upload_ids(self, ids: Sequence[int]) -> int:
        n = len(ids)
        self.ids_host[:n] = torch.as_tensor(ids, dtype=torch.int32)
        self.ids_dev[:n].copy_(self.ids_host[:n], non_blocking=True)
        return self.ids_dev.data_ptr()

    def timing(self) -> native.Timing:
        t = native.Timing()
        native.check("sr_last_timing", self.lib.sr_last_timing(self.handle, C.byref(t)))
        return t


@dataclass
class EngineStats:
    """Device-side accounting of every native call (CUDA-event times from
    ``sr_last_timing``, our kernel launches, host<->device bytes)."""

    calls: int = 0
    prefill_ms: float = 0.0
    decode_ms: float = 0.0
    prefill_tokens: int = 0
    decode_tokens: int = 0      # tokens produced by the decode graph (n_gen - 1)
    decode_bytes: float = 0.0   # algorithmic HBM bytes of those decode steps
    prefill_bytes: float = 0.0  # algorithmic HBM bytes of the prefill passes (+ LM head)
    prefill_flops: float = 0.0
    launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def _prefill_launches(self, spec, n: int, max_tokens: int = 256) -> int:
        chunks = -(-n // max_tokens)
        return chunks * (1 + 9 * spec.n_layers)

    def add_generate(self, m: "DeviceModel", n_ids: int, n_gen: int, start: int) -> None:
        t = m.timing()
        spec = m.spec
        self.calls += 1
        self.prefill_ms += t.prefill_ms
        self.decode_ms += t.decode_ms
        if t.prefill_tokens == 0:  # one fed token: every new token is a decode step
            steps = n_gen
            self.decode_tokens += steps
            for i in range(steps):
                self.decode_bytes += spec.decode_bytes(start + i)
            self.launches += 2  # decode_begin + the persistent decode kernel
        else:
            self.prefill_tokens += n_ids
            steps = max(0, n_gen - 1)
            self.decode_tokens += steps
            b, f = spec.prefill_cost(start, n_ids, 1, m.max_tokens)
            self.prefill_bytes += b
            self.prefill_flops += f
            ctx0 = start + n_ids
            for i in range(steps):
                self.decode_bytes += spec.decode_bytes(ctx0 + i)
            # decode_begin + prefill + first-token LM head + one persistent
            # decode kernel for the whole step (decode_mk.cu)
            self.launches += self._prefill_launches(spec, n_ids) + 3
        self.h2d_bytes += 4 * n_ids + 64
        self.d2h_bytes += 4 * (2 + m.max_new) * 2

    def add_score(self, m: "DeviceModel", n_ids: int, start: int, head_rows: int = 1) -> None:
        t = m.timing()
        b, f = m.spec.prefill_cost(start, n_ids, head_rows, m.max_tokens)
        self.prefill_bytes += b
        self.prefill_flops += f
        self.calls += 1
        self.prefill_ms += t.prefill_ms
        self.prefill_tokens += n_ids
        self.launches += self._prefill_launches(m.spec, n_ids) + 2
        self.h2d_bytes += 4 * n_ids + 64
        self.d2h_bytes += 16

    def add_pass(self, spec, starts, counts) -> None:
        """Algorithmic cost of one multi-sequence pass: the weights stream
        once for every row, each sequence reads its own context."""
        kvb = spec.kv_bytes_per_token()
        attn = 4 * spec.n_layers * spec.n_heads * spec.head_dim
        rows = sum(counts)
        self.prefill_bytes += 2 * (spec.body_params() + spec.head_params())
        self.prefill_flops += 2 * rows * spec.body_params() + 2 * len(counts) * spec.head_params()
        for s0, n in zip(starts, counts):
            self.prefill_bytes += (s0 + 2 * n) * kvb
            self.prefill_flops += attn * n * (s0 + n / 2)

    def snapshot(self) -> "EngineStats":
        return EngineStats(**self.__dict__)

    def minus(self, other: "EngineStats") -> "EngineStats":
        return EngineStats(**{k: getattr(self, k) - getattr(other, k) for k in self.__dict__})

    def plus(self, other: "EngineStats") -> "EngineStats":
        return EngineStats(**{k: getattr(self, k) + getattr(other, k) for k in self.__dict__})


@dataclass
class _Pages:
    pages: list[int]
    table_dev: torch.Tensor
    table_host: torch.Tensor
    synced: int = 0  # entries already uploaded


class NativeEngine:
    """``host.DeviceEngine`` over a ``DeviceModel``."""

    # several streams' fresh rows share one device pass (sr_score_batch): a
    # scoring call extends the generation stream in the same pass
    multi_span_passes = True

    def __init__(self, model: DeviceModel, vocab: Vocab) -> None:
        self.model = model
        self.spec = model.spec
        self.vocab = vocab
        self.streams: list[Stream] = []
        self._classes: dict[tuple[str, ...], torch.Tensor] = {}
        # token-indexed tables span the global vocabulary (the embedding rows)
        self.n_ids = model.spec.embed_rows or model.spec.vocab_rows
        self.first_digit = first_digit_table(vocab, self.n_ids).to(model.device)
        self.max_pages = math.ceil(model.max_pos / PAGE)
        self.last_margins: list[float] = []
        self.stats = EngineStats()

    # -- page management -------------------------------------------------
    def attach(self, stream: Stream) -> None:
        stream.handle = _Pages(
            pages=[],
            table_dev=torch.zeros(self.max_pages, dtype=torch.int32, device=self.model.device),
            table_host=torch.zeros(self.max_pages, dtype=torch.int32, pin_memory=True))
        self.streams.append(stream)

    def truncate(self, stream: Stream, keep: int) -> None:
        del stream.ids[keep:]
        pg: _Pages = stream.handle
        need = math.ceil(keep / PAGE)
        while len(pg.pages) > need:
            self.model.free_pages.append(pg.pages.pop())
        pg.synced = min(pg.synced, len(pg.pages))

    def _ensure(self, stream: Stream, n_positions: int, protect=()) -> None:
        if n_positions > self.model.max_pos:
            raise ValueError(f"context of {n_positions} positions exceeds max_pos "
                             f"{self.model.max_pos}")
        pg: _Pages = stream.handle
        need = math.ceil(n_positions / PAGE)
        free = self.model.free_pages
        while len(pg.pages) < need:
            if not free:
                busy = getattr(self, "busy", ())
                victims = sorted((s for s in self.streams if s is not stream and s not in protect
                                  and s not in busy and s.handle.pages),
                                 key=lambda s: s.stamp)
                if not victims:
                    raise MemoryError("K/V page pool exhausted")
                self.truncate(victims[0], 0)
                continue
            pg.pages.append(free.pop())
        if pg.synced < len(pg.pages):
            lo, hi = pg.synced, len(pg.pages)
            pg.table_host[lo:hi] = torch.as_tensor(pg.pages[lo:hi], dtype=torch.int32)
            pg.table_dev[lo:hi].copy_(pg.table_host[lo:hi], non_blocking=True)
            pg.synced = hi

    def _class_table(self, stop: tuple[str, ...]) -> torch.Tensor:
        t = self._classes.get(stop)
        if t is None:
            cls = self.vocab.token_classes(stop, self.n_ids)
            t = torch.from_numpy(cls.copy()).to(self.model.device)
            self._classes[stop] = t
        return t

    # -- engine calls ----------------------------------------------------
    def generate(self, stream: Stream, suffix: Sequence[int], max_new: int,
                 stop: tuple[str, ...]) -> tuple[list[int], int]:
        """Greedy generation of up to ``max_new`` tokens.  A request longer
        than one native call allows (``max_new`` of the model) continues in
        further ``sr_generate`` calls fed the last token, so every path honours
        ``request.max_tokens`` exactly."""
        gen, finish = self._generate_once(stream, suffix, max_new, stop)
        margins = list(self.last_margins)
        while finish == 0 and len(gen) < max_new:  # FINISH_LENGTH at the call cap
            more, finish = self._generate_once(stream, gen[-1:], max_new - len(gen), stop)
            gen.extend(more)
            margins.extend(self.last_margins)
        self.last_margins = margins
        return gen, finish

    def _generate_once(self, stream: Stream, suffix: Sequence[int], max_new: int,
                       stop: tuple[str, ...]) -> tuple[list[int], int]:
        m = self.model
        max_new = min(max_new, m.max_new)
        start = len(stream.ids)
        self._ensure(stream, start + len(suffix) + max_new)
        cls = self._class_table(stop)
        ids_ptr = m.upload_ids(suffix)
        native.check("sr_generate", m.lib.sr_generate(
            m.handle, C.c_void_p(stream.handle.table_dev.data_ptr()), start,
            C.c_void_p(ids_ptr), len(suffix), max_new, C.c_void_p(cls.data_ptr()),
            C.c_void_p(m.out_dev.data_ptr()), C.c_void_p(m.margin_dev.data_ptr()),
            m.stream_ptr))
        m.out_host.copy_(m.out_dev, non_blocking=True)
        m.margin_host.copy_(m.margin_dev, non_blocking=True)
        torch.cuda.current_stream(m.device).synchronize()
        n, finish = int(m.out_host[0]), int(m.out_host[1])
        gen = m.out_host[2:2 + n].tolist()
        self.last_margins = m.margin_host[:n].tolist()
        self.stats.add_generate(m, len(suffix), n, start)
        stream.ids.extend(suffix)
        stream.ids.extend(gen[:-1])
        return gen, finish

    def score(self, stream: Stream, suffix: Sequence[int], threshold: int) -> Readout:
        m = self.model
        start = len(stream.ids)
        self._ensure(stream, start + len(suffix))
        ids_ptr = m.upload_ids(suffix)
        native.check("sr_score", m.lib.sr_score(
            m.handle, C.c_void_p(stream.handle.table_dev.data_ptr()), start,
            C.c_void_p(ids_ptr), len(suffix), C.c_void_p(self.first_digit.data_ptr()),
            int(threshold), C.c_void_p(m.readout_dev.data_ptr()), m.stream_ptr))
        m.readout_host.copy_(m.readout_dev, non_blocking=True)
        torch.cuda.current_stream(m.device).synchronize()
        self.stats.add_score(m, len(suffix), start)
        stream.ids.extend(suffix)
        r = m.readout_host
        margin = r[2:3].view(torch.float32).item()
        return Readout(score=int(r[0]), accept=bool(int(r[1])), flags=0, margin=margin,
                       argmax=int(r[3]))

    # -- multi-sequence passes ----------------------------
    def _batch(self, streams: Sequence[Stream], suffixes: Sequence[Sequence[int]],
               room: int = 0):
        """Stage one multi-sequence pass: pages for every stream (no stream of
        the batch is evicted for another), the ids back to back, and the
        (position, page) of every row."""
        m = self.model
        if len(set(id(s) for s in streams)) != len(streams):
            raise ValueError("a batched pass needs distinct streams")
        starts, counts, meta, flat = [], [], [], []
        for st, suf in zip(streams, suffixes):
            start = len(st.ids)
            self._ensure(st, start + len(suf) + room, protect=streams)
            pages = st.handle.pages
            for i in range(len(suf)):
                meta += [start + i, pages[(start + i) // PAGE]]
            starts.append(start)
            counts.append(len(suf))
            flat.extend(suf)
        n = len(streams)
        ids_ptr = m.upload_ids(flat)
        k = len(meta)
        m.meta_host[:k] = torch.as_tensor(meta, dtype=torch.int32)
        m.meta_dev[:k].copy_(m.meta_host[:k], non_blocking=True)
        meta_dev = m.meta_dev
        tables = (C.c_void_p * n)(*[st.handle.table_dev.data_ptr() for st in streams])
        return (n, tables, (C.c_int32 * n)(*starts), (C.c_int32 * n)(*counts),
                C.c_void_p(ids_ptr), meta_dev, len(flat))

    def _passes(self, lengths: Sequence[int]) -> list[list[int]]:
        """Group sequences (in order) into passes of at most max_tokens rows."""
        cap = self.model.max_tokens
        out, cur, rows = [], [], 0
        for i, n in enumerate(lengths):
            if cur and rows + n > cap:
                out.append(cur)
                cur, rows = [], 0
            cur.append(i)
            rows += n
        if cur:
            out.append(cur)
        return out

    def score_batch(self, streams: Sequence[Stream], suffixes: Sequence[Sequence[int]],
                    threshold: int) -> list[Readout]:
        """``score`` for several streams, as few passes (``sr_score_batch``)
        as max_tokens rows allow; a sequence longer than that alone takes the
        chunked single-sequence path."""
        res: list[Readout | None] = [None] * len(streams)
        for group in self._passes([len(s) for s in suffixes]):
            if len(group) == 1 and len(suffixes[group[0]]) > self.model.max_tokens:
                i = group[0]
                res[i] = self.score(streams[i], suffixes[i], threshold)
                continue
            sub = self._score_pass([streams[i] for i in group], [suffixes[i] for i in group],
                                   threshold)
            for i, r in zip(group, sub):
                res[i] = r
        return res

    def _score_pass(self, streams, suffixes, threshold: int) -> list[Readout]:
        m = self.model
        n, tables, starts, counts, ids, meta_dev, rows = self._batch(streams, suffixes)
        out = m.batch_out
        native.check("sr_score_batch", m.lib.sr_score_batch(
            m.handle, n, tables, starts, counts, ids, C.c_void_p(meta_dev.data_ptr()),
            C.c_void_p(self.first_digit.data_ptr()), int(threshold), C.c_void_p(out.data_ptr()),
            m.stream_ptr))
        host = out[:4 * n].cpu()
        self.stats.calls += 1
        self.stats.prefill_ms += m.timing().prefill_ms
        self.stats.prefill_tokens += rows
        self.stats.add_pass(self.spec, list(starts), list(counts))
        self.stats.launches += 9 * self.spec.n_layers + 3 + n
        self.stats.h2d_bytes += 12 * rows
        self.stats.d2h_bytes += 16 * n
        res = []
        for i, (st, suf) in enumerate(zip(streams, suffixes)):
            st.ids.extend(suf)
            r = host[4 * i:4 * i + 4]
            res.append(Readout(score=int(r[0]), accept=bool(int(r[1])), flags=0,
                               margin=r[2:3].view(torch.float32).item(), argmax=int(r[3])))
        return res

    def step_batch(self, streams: Sequence[Stream], feeds: Sequence[Sequence[int]],
                   room: int = 0) -> list[int]:
        """One greedy token for each stream after feeding ``feeds[i]`` (prompt
        rows or the previous token), in as few ``sr_step_batch`` passes as
        max_tokens allows; the fed tokens are committed to the streams.
        ``room`` positions are reserved past the feed for later tokens."""
        m = self.model
        feeds = [list(f) for f in feeds]
        for i, f in enumerate(feeds):  # beyond one pass: all but the last token on the chunked path
            if len(f) > m.max_tokens:
                self.prefill(streams[i], f[:-1])
                feeds[i] = f[-1:]
        out, margins = m.batch_out, m.batch_margins
        toks: list[int] = [0] * len(streams)
        for group in self._passes([len(f) for f in feeds]):
            n, tables, starts, counts, ids, meta_dev, rows = self._batch(
                [streams[i] for i in group], [feeds[i] for i in group], room=room)
            native.check("sr_step_batch", m.lib.sr_step_batch(
                m.handle, n, tables, starts, counts, ids, C.c_void_p(meta_dev.data_ptr()),
                C.c_void_p(out.data_ptr()), C.c_void_p(margins.data_ptr()), m.stream_ptr))
            for i, t in zip(group, out[:n].tolist()):
                toks[i] = t
            self.stats.calls += 1
            self.stats.prefill_ms += m.timing().prefill_ms
            self.stats.prefill_tokens += rows
            self.stats.add_pass(self.spec, list(starts), list(counts))
            self.stats.launches += 9 * self.spec.n_layers + 3
            self.stats.h2d_bytes += 12 * rows
            self.stats.d2h_bytes += 4 * n
        for st, f in zip(streams, feeds):
            st.ids.extend(f)
        return toks

    def generate_batch(self, streams: Sequence[Stream], suffixes: Sequence[Sequence[int]],
                       max_new: int, stop: tuple[str, ...]) -> list[tuple[list[int], int]]:
        """Greedy ``generate`` for several streams, one batched step per token
        (``step_batch``): each step streams the weights once for every live
        sequence.  Finished sequences leave the batch."""
        from .host import finish_of

        classes = self.vocab.token_classes(stop, self.n_ids)
        live = list(range(len(streams)))
        gens: list[list[int]] = [[] for _ in streams]
        feed = [list(s) for s in suffixes]
        self.last_margins = []
        while live:
            toks = self.step_batch([streams[i] for i in live], [feed[i] for i in live], room=max_new)
            nxt = []
            for k, i in enumerate(live):
                gens[i].append(toks[k])
                if classes[toks[k]] in (CLASS_STOP, CLASS_END_THINK) or len(gens[i]) >= max_new:
                    continue
                feed[i] = [toks[k]]
                nxt.append(i)
            live = nxt
        return [(g, finish_of(g, classes)) for g in gens]

    def prefill(self, stream: Stream, suffix: Sequence[int]) -> None:
        """Commit ``suffix`` to the stream's K/V (no token is chosen)."""
        self.forward_logits(stream, suffix, all_rows=False)

    def verify_tokens(self, stream: Stream, suffix: Sequence[int]) -> tuple[list[int], list[float]]:
        """Prefill ``suffix`` and return the greedy choice after every fed
        token (token-level speculation, ``sr_verify_tokens``)."""
        m = self.model
        start = len(stream.ids)
        n = len(suffix)
        self._ensure(stream, start + n)
        ids_ptr = m.upload_ids(suffix)
        native.check("sr_verify_tokens", m.lib.sr_verify_tokens(
            m.handle, C.c_void_p(stream.handle.table_dev.data_ptr()), start, C.c_void_p(ids_ptr), n,
            C.c_void_p(m.out_dev.data_ptr()), C.c_void_p(m.margin_dev.data_ptr()), m.stream_ptr))
        m.out_host[:n].copy_(m.out_dev[:n], non_blocking=True)
        m.margin_host[:n].copy_(m.margin_dev[:n], non_blocking=True)
        torch.cuda.current_stream(m.device).synchronize()
        self.stats.add_score(m, n, start, head_rows=n)
        stream.ids.extend(suffix)
        return m.out_host[:n].tolist(), m.margin_host[:n].tolist()

    def forward_logits(self, stream: Stream, suffix: Sequence[int], all_rows: bool = True) -> torch.Tensor:
        """Test hook: prefill ``suffix`` and return fp32 logits (device)."""
        m = self.model
        start = len(stream.ids)
        self._ensure(stream, start + len(suffix))
        ids_ptr = m.upload_ids(suffix)
        rows = len(suffix) if all_rows else 1
        out = torch.empty(rows, self.spec.vocab_rows, dtype=torch.float32, device=m.device)
        native.check("sr_forward_logits", m.lib.sr_forward_logits(
            m.handle, C.c_void_p(stream.handle.table_dev.data_ptr()), start,
            C.c_void_p(ids_ptr), len(suffix), 1 if all_rows else 0,
            C.c_void_p(out.data_ptr()), m.stream_ptr))
        torch.cuda.current_stream(m.device).synchronize()
        stream.ids.extend(suffix)
        return out


class PeerTransport:
    """This rank's NVLink peer-memory exchange buffer (``sr_tp_peer_*``): the
    transport of the fused tensor-parallel decode kernel and of the one-shot
    prefill / readout collectives.  Ranks connect through CUDA IPC handles
    (``connect_ipc``, across processes) or plain device pointers
    (``connect_local``, ranks of one process)."""

    # mailboxes sized for the bench shapes: d_model <= 8192, 256-row prefill chunks
    DEC_ROW = 8192
    MAX_ELEMS = 256 * 8192

    def __init__(self, rank: int, world: int, max_elems: int = MAX_ELEMS,
                 dec_row: int = DEC_ROW) -> None:
        self.lib = native.load()
        self.rank, self.world = rank, world
        h = C.c_void_p()
        native.check("sr_tp_peer_create", self.lib.sr_tp_peer_create(world, rank, max_elems,
                                                                     dec_row, C.byref(h)))
        self.handle = h

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        native.check("sr_tp_peer_handle", self.lib.sr_tp_peer_handle(self.handle, buf))
        return bytes(buf)

    def connect_ipc(self, handles: list[bytes]) -> None:
        buf = (C.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(handles))
        native.check("sr_tp_peer_open", self.lib.sr_tp_peer_open(self.handle, buf))

    def base(self) -> int:
        v = C.c_uint64()
        native.check("sr_tp_peer_base", self.lib.sr_tp_peer_base(self.handle, C.byref(v)))
        return v.value

    def connect_local(self, bases: list[int]) -> None:
        arr = (C.c_uint64 * self.world)(*bases)
        native.check("sr_tp_peer_attach", self.lib.sr_tp_peer_attach(self.handle, arr))

    def close(self) -> None:
        if self.handle is not None and self.handle.value:
            self.lib.sr_tp_peer_destroy(self.handle)
            self.handle = None


class TensorParallel:
    """One rank of a tensor-parallel base model (config C4): the rank / world
    plus its transports -- an NCCL communicator of the C-ABI
    (``sr_tp_comm_create``), a ``PeerTransport``, or both (then prefill uses
    NCCL's ring all-reduce and decode the fused peer-memory kernel)."""

    def __init__(self, rank: int, world: int, uid: bytes | None = None,
                 peer: PeerTransport | None = None) -> None:
        self.rank, self.world = rank, world
        self.comm = None
        self.peer = peer
        if uid is not None:
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            comm = C.c_void_p()
            native.check("sr_tp_comm_create",
                         native.load().sr_tp_comm_create(buf, world, rank, C.byref(comm)))
            self.comm = comm

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        native.check("sr_tp_unique_id", native.load().sr_tp_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_dist(cls, group=None, transport: str = "peer") -> "TensorParallel":
        """Collective over an initialised torch.distributed group (gloo or
        nccl): ``transport`` "peer" (NVLink peer memory, IPC handles
        all-gathered), "nccl", or "both"."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = peer = None
        if transport in ("nccl", "both"):
            box = [cls.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = box[0]
        if transport in ("peer", "both"):
            peer = PeerTransport(rank, world)
            handles: list = [None] * world
            dist.all_gather_object(handles, peer.ipc_handle(), group=group)
            peer.connect_ipc(handles)
        return cls(rank, world, uid, peer)

    @classmethod
    def single(cls) -> "TensorParallel":
        """World-size-1 NCCL communicator: runs every TP code path on one GPU."""
        return cls(0, 1, cls.unique_id())

    @classmethod
    def local_group(cls, world: int) -> list["TensorParallel"]:
        """``world`` ranks in this process over peer memory (e.g. several
        ranks sharing one GPU in a test): buffers connected by pointer."""
        peers = [PeerTransport(r, world) for r in range(world)]
        bases = [p.base() for p in peers]
        for p in peers:
            p.connect_local(bases)
        return [cls(r, world, None, peers[r]) for r in range(world)]

    def close(self) -> None:
        if self.comm is not None and self.comm.value:
            native.load().sr_tp_comm_destroy(self.comm)
            self.comm = None
        if self.peer is not None:
            self.peer.close()
            self.peer = None


class B200Backend(ModelBackend):
    """Drop-in ``Backend`` whose model runs on the B200 (see module doc)."""

    def __init__(self, spec: ModelSpec | str, role: BackendRole, *, seed: int = 0,
                 weights: dict[str, torch.Tensor] | None = None, max_ctx: int = 8192,
                 n_streams: int = 4, threshold: int = 7, max_new: int = 256,
                 max_tokens: int = 256, device: str = "cuda", init_device: str | None = None,
                 vocab: Vocab | None = None, types=None, record: bool = False,
                 tp: "TensorParallel | None" = None, decode_layout: bool = True) -> None:
        """``decode_layout``: keep the decode kernel's tile-major copy of the
        streamed weights (``decode_tiles``; ~8 % faster decode for the 32B at
        the cost of holding those weights twice); False streams the row-major
        weights through TMA boxes with CUDA-core GEMVs."""
        if not torch.cuda.is_available():
            raise RuntimeError("B200Backend needs a CUDA device (no CPU fallback)")
        spec = get_spec(spec) if isinstance(spec, str) else spec
        full_spec = spec
        if tp is not None:  # this rank's shard of the model (config C4)
            spec = tp_spec(full_spec, tp.rank, tp.world)
        if weights is None:
            init_device = init_device or ("cpu" if spec.d_model <= 512 else device)
            if tp is not None:
                weights = make_tp_weights(full_spec, tp.rank, tp.world, seed, device=init_device)
            else:
                weights = make_weights(spec, seed, device=init_device)
        elif tp is not None and tuple(weights["lm_head"].shape)[0] == full_spec.vocab_rows:
            weights = shard_weights(weights, full_spec, tp.rank, tp.world)
        max_pos = max_ctx + max_new + 64
        pages_per_stream = math.ceil(max_pos / PAGE) + 1
        model = DeviceModel(spec, weights, max_pos=max_pos, n_pages=n_streams * pages_per_stream,
                            max_tokens=max_tokens, max_new=max_new, device=device,
                            decode_layout=decode_layout)
        if tp is not None and tp.comm is not None:
            native.check("sr_model_set_tp", model.lib.sr_model_set_tp(model.handle, tp.comm))
        if tp is not None and tp.peer is not None:
            native.check("sr_model_set_tp_peer",
                         model.lib.sr_model_set_tp_peer(model.handle, tp.peer.handle))
        self.tp = tp
        vocab = vocab or shared_vocab(spec.vocab_text)
        T = types
        prof_cls = T.BackendProfile if T else BackendProfile
        role_cls = T.BackendRole if T else BackendRole
        profile = prof_cls(name=f"b200-{spec.name}", role=role_cls(role.value),
                           decode_s_per_token=spec.decode_bytes(0) / 6.4e12,
                           prefill_tokens_per_s=1e4)
        self.device_model = model
        engine = NativeEngine(model, vocab)
        if tp is not None:  # sr_score_batch / sr_step_batch are single-rank: no multi-span passes
            engine.multi_span_passes = False
        super().__init__(engine, vocab, profile, n_streams=n_streams,
                         threshold=threshold, types=types, record=record)


def build_pair(pair: str = "tiny", *, seed: int = 0, max_ctx: int = 8192, threshold: int = 7,
               types=None, record: bool = False, base_tp: TensorParallel | None = None,
               **kw) -> tuple[B200Backend, B200Backend]:
    """(small, base) backends for a named model pair (``shapes.PAIRS``).
    With ``base_tp`` the base model is this rank's tensor-parallel shard and
    the draft is replicated (SPMD: every rank drives the same trajectory)."""
    small_name, base_name = PAIRS[pair]
    small = B200Backend(small_name, BackendRole.SMALL, seed=seed, max_ctx=max_ctx,
                        threshold=threshold, types=types, record=record, **kw)
    base = B200Backend(base_name, BackendRole.BASE, seed=seed, max_ctx=max_ctx,
                       threshold=threshold, types=types, record=record, tp=base_tp, **kw)
    return small, base
