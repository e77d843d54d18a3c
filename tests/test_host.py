"""Host logic: vocabulary / token model, stream pool, prompt cache, C-ABI
symbol table, model shapes -- everything the device path relies on that can
be checked without a GPU."""

import ctypes
import re

import numpy as np
import pytest
import torch

from paper_2504_07891_b200 import domain
from paper_2504_07891_b200.host import StreamPool, _PromptCache, common_prefix, finish_of
from paper_2504_07891_b200.shapes import (MODELS, get_spec, gu_interleave, gu_split, make_tensor,
                                          make_weights, rope_table, tensor_shapes)
from paper_2504_07891_b200.vocab import (CLASS_END_THINK, CLASS_MASKED, CLASS_PLAIN, CLASS_STOP,
                                         END_THINK_ID, JUDGE_CUE_ID, Vocab, shared_vocab)


# ------------------------------------------------------------------ vocab --
def test_render_encode_round_trip(tiny_vocab):
    rng = np.random.default_rng(0)
    for _ in range(50):
        ids = rng.integers(0, tiny_vocab.n_text, size=int(rng.integers(1, 200))).tolist()
        text = tiny_vocab.render(ids)
        assert tiny_vocab.encode(text) == ids
        assert domain.count_tokens(text) == len(ids)


def test_concatenated_renderings_never_fuse(tiny_vocab):
    a, b = [20, 21, 22], [30, 31]
    assert tiny_vocab.encode(tiny_vocab.render(a) + tiny_vocab.render(b)) == a + b


def test_unknown_words_hash_into_ordinary_range(tiny_vocab):
    lo, hi = tiny_vocab.ordinary_range()
    for w in ("You", "grading", "w3</think>", "0-9", "é"):
        i = tiny_vocab.word_id(w)
        assert lo <= i < hi
        assert tiny_vocab.word_id(w) == i  # stable


def test_special_ids(tiny_vocab):
    assert tiny_vocab.encode("0 9 <think> </think> 0-9:") == [0, 9, 10, END_THINK_ID, JUDGE_CUE_ID]
    tmpl = domain.render_verification_prompt("p", "c", "x")
    assert tiny_vocab.encode(tmpl)[-1] == JUDGE_CUE_ID  # the judge cue is the last token


def test_boundary_density_and_stop_classes(tiny_vocab):
    cls = tiny_vocab.token_classes(domain.DEFAULT_STEP_STOP_MARKERS, 4096 + 64)
    n_stop = int((cls == CLASS_STOP).sum())
    assert 4096 / 24 * 0.7 < n_stop < 4096 / 24 * 1.3
    assert cls[END_THINK_ID] == CLASS_END_THINK
    assert (cls[4096:] == CLASS_MASKED).all()
    for i in np.nonzero(cls == CLASS_STOP)[0][:50]:
        assert tiny_vocab.render_one(int(i)).endswith("\n")
    no_stop = tiny_vocab.token_classes((), 4096)
    assert set(np.unique(no_stop)) <= {CLASS_PLAIN, CLASS_END_THINK}


def test_problem_generator_deterministic(tiny_vocab):
    p = tiny_vocab.problem(64, 3)
    assert p == tiny_vocab.problem(64, 3) and domain.count_tokens(p) == 64
    assert p != tiny_vocab.problem(64, 4)


def test_full_vocab_words_unique():
    v = Vocab(151_936)
    assert len(set(v.words)) == v.n_text


# ----------------------------------------------------------- stream logic --
def test_common_prefix():
    rng = np.random.default_rng(1)
    for _ in range(300):
        a = rng.integers(0, 5, size=int(rng.integers(0, 60))).tolist()
        b = a[: int(rng.integers(0, len(a) + 1))] + rng.integers(0, 5, size=int(rng.integers(0, 10))).tolist()
        want = 0
        while want < min(len(a), len(b)) and a[want] == b[want]:
            want += 1
        assert common_prefix(a, b) == want


def test_stream_pool_prefers_longest_prefix_then_lru():
    pool = StreamPool(3)
    s, keep = pool.acquire([1, 2, 3])
    assert keep == 0
    s.ids = [1, 2, 3, 4]
    t, keep = pool.acquire([1, 2, 3, 4, 5])
    assert t is s and keep == 4
    t, keep = pool.acquire([1, 2, 3, 4])
    assert t is s and keep == 3  # the last prompt token is always recomputed
    u, keep = pool.acquire([9, 9])
    assert u is not s and keep == 0


def test_prompt_cache_incremental_equals_full(tiny_vocab):
    pc = _PromptCache(tiny_vocab)
    base = tiny_vocab.render(list(range(16, 80)))
    assert pc.encode(base) == tiny_vocab.encode(base)
    longer = base + tiny_vocab.render([100, 101]) + "kab"
    assert pc.encode(longer) == tiny_vocab.encode(longer)
    assert pc.encode(base + "</think>\n") == tiny_vocab.encode(base + "</think>\n")


def test_finish_codes():
    cls = np.zeros(10, np.uint8)
    cls[3], cls[4] = CLASS_STOP, CLASS_END_THINK
    assert finish_of([1, 3], cls) == 1
    assert finish_of([1, 4], cls) == 2
    assert finish_of([1, 2], cls) == 0


# ---------------------------------------------------------------- shapes --
def test_param_counts_match_public_cards():
    # P_body 1.310 B / 6.526 B / 31.21 B
    assert abs(get_spec("r1-1.5b").body_params() / 1e9 - 1.310) < 0.01
    assert abs(get_spec("qwen2.5-7b").body_params() / 1e9 - 6.526) < 0.01
    assert abs(get_spec("qwq-32b").body_params() / 1e9 - 31.21) < 0.02
    assert get_spec("qwq-32b").kv_bytes_per_token() == 262_144


def test_gate_up_interleave_round_trip():
    g, u = torch.randn(64, 8), torch.randn(64, 8)
    w = gu_interleave(g, u)
    assert torch.equal(w[:16], g[:16]) and torch.equal(w[16:32], u[:16])
    g2, u2 = gu_split(w)
    assert torch.equal(g, g2) and torch.equal(u, u2)


def test_weights_deterministic_and_sliceable():
    spec = get_spec("tiny-base")
    a = make_weights(spec, 0)
    b = make_weights(spec, 0, layers=[2])
    assert set(b) == {k for k in a if not k.startswith("layers.") or k.startswith("layers.2.")}
    assert torch.equal(a["layers.2.wqkv"], b["layers.2.wqkv"])
    assert not torch.equal(a["layers.1.wqkv"], a["layers.2.wqkv"])
    for name, shape in tensor_shapes(spec).items():
        assert tuple(a[name].shape) == shape and a[name].dtype == torch.bfloat16


def test_judge_circuit_present_only_in_base():
    base, draft = get_spec("tiny-base"), get_spec("tiny-draft")
    e = make_tensor(base, 0, "embed").float()
    assert e[JUDGE_CUE_ID].norm() > 10 * e[100].norm()
    e2 = make_tensor(draft, 0, "embed").float()
    assert e2[JUDGE_CUE_ID].norm() < 3 * e2[100].norm()


def test_rope_table():
    t = rope_table(get_spec("tiny-base"), 100)
    assert t.shape == (100, 64, 2)
    assert torch.allclose(t[0, :, 0], torch.ones(64)) and torch.allclose(t[0, :, 1], torch.zeros(64))


# ----------------------------------------------------------------- C-ABI --
def test_cabi_library_exports_every_header_symbol():
    """The built library loads on a CPU box and exports every function the
    header declares (no compute calls without a GPU)."""
    from paper_2504_07891_b200 import native

    header = (native.LIB_PATH.parents[1] / "include" / "specreason_b200.h").read_text()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(sr_\w+)\s*\(", header, flags=re.M))
    assert declared == set(native.EXPORTS), declared ^ set(native.EXPORTS)
    lib = native.load()
    for name in declared:
        assert hasattr(lib, name)
    assert lib.sr_abi_version() == 1
    assert ctypes.sizeof(native.Readout) == 16


def test_cabi_rejects_bad_descriptor():
    from paper_2504_07891_b200 import native

    lib = native.load()
    d = native.ModelDesc(n_layers=1, d_model=100, n_heads=1, n_kv_heads=1, head_dim=128,
                         d_ffn=64, vocab_rows=16, vocab_text=16, rms_eps=1e-6, max_pos=8,
                         max_tokens=4, max_new=4, n_pages=1)
    assert lib.sr_workspace_bytes(ctypes.byref(d)) == 0
    assert b"d_model" in lib.sr_last_error()


def test_native_errors_map_onto_the_reference_hierarchy(tiny_vocab):
    """Device failures surface as BackendMisbehavior (collectives as
    TransportError), so the engine adds the step context (engine.py:269-273)."""
    import pytest

    from paper_2504_07891_b200 import contract
    from paper_2504_07891_b200.contract import GenerationRequest, VerificationRequest
    from paper_2504_07891_b200.domain import BackendProfile, BackendRole
    from paper_2504_07891_b200.host import ModelBackend
    from paper_2504_07891_b200.native import NativeError

    class Failing:
        spec = None

        def __init__(self, code):
            self.code = code

        def attach(self, stream):
            stream.handle = None

        def truncate(self, stream, keep):
            del stream.ids[keep:]

        def generate(self, *a):
            raise NativeError("sr_generate", self.code, "boom")

        def score(self, *a):
            raise NativeError("sr_score", self.code, "boom")

    prof = BackendProfile(name="x", role=BackendRole.BASE, decode_s_per_token=1e-3,
                          prefill_tokens_per_s=1e3)
    b = ModelBackend(Failing(700), tiny_vocab, prof)
    with pytest.raises(contract.BackendMisbehavior):
        b.generate_step(GenerationRequest(prompt="a b ", max_tokens=4))
    t = ModelBackend(Failing(1004), tiny_vocab, prof)
    with pytest.raises(contract.TransportError):
        t.score_step(VerificationRequest("a", "b ", "c "))


def test_decode_tiles_layout():
    """The decode kernel's tile-major weight copy (``backend.decode_tiles``,
    ``sr_model_set_decode_tiles``): tile (b, k) = rows 32b.. x columns k*tc..
    in (b, k) order, each as tc/64 boxes of [32][64] whose 16-B chunk j of
    row r sits at chunk position j ^ (r & 7)."""
    import torch

    from paper_2504_07891_b200.backend import decode_tiles

    for N, K in ((64, 512), (96, 128), (32, 256), (32, 768)):
        w = torch.randn(N, K).to(torch.bfloat16)
        tc = min(K, 256)
        t = decode_tiles(w).view(N // 32, K // tc, tc // 64, 32, 8, 8)
        b, r, c = torch.meshgrid(torch.arange(N // 32), torch.arange(32), torch.arange(K), indexing="ij")
        k, cc = c // tc, c % tc
        got = t[b, k, cc // 64, r, ((cc % 64) // 8) ^ (r & 7), cc % 8]
        assert torch.equal(got, w.view(N // 32, 32, K))
    with pytest.raises(ValueError):
        decode_tiles(torch.zeros(48, 256, dtype=torch.bfloat16))  # rows not a multiple of 32
