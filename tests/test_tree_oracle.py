"""The layer-streamed prefix-tree oracle (``oracle/tree_oracle.py``) computes
the same function as ``RefModel`` (CPU, tiny shapes), and its prefix tree
gives each position exactly its own sequence's context."""

import pytest
import torch

from oracle.ref_model import RefModel
from oracle.tree_oracle import PrefixTrie, TreeOracle, choice_summary, readout_ambiguity
from paper_2504_07891_b200.shapes import get_spec, make_weights


def _seqs(n_text, seed=0):
    g = torch.Generator().manual_seed(seed)
    r = lambda n: torch.randint(16, n_text, (n,), generator=g).tolist()  # noqa: E731
    trunk = r(70)
    return [trunk + r(20), trunk[:40] + r(30), trunk + r(20)[:5], trunk[:40], r(12), trunk + r(3)]


def test_trie_layout():
    t = PrefixTrie()
    seqs = [[1, 2, 3, 4], [1, 2, 5], [1, 2, 3], [7]]
    for s in seqs:
        t.insert(s)
    t.finalize()
    assert t.n_slots == 6  # 1 2 | 3 4 | 5 | 7 -> shared prefix stored once
    ids, pos, din, dout = t.slot_tables()
    for k, s in enumerate(seqs):
        for p_, tok in enumerate(s):
            sl = t.slot_of(k, p_)
            assert int(ids[sl]) == tok and int(pos[sl]) == p_


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("name", ["tiny-draft", "tiny-base"])
def test_tree_oracle_equals_refmodel(name, exact):
    spec = get_spec(name)
    w = make_weights(spec, 0)
    seqs = _seqs(spec.vocab_text)
    trie = PrefixTrie()
    for s in seqs:
        trie.insert(s)
    tor = TreeOracle(spec, lambda n: w[n], exact_fp32=exact)
    hid = tor.hidden(trie)
    ref = RefModel(spec, w, exact_fp32=exact)
    worst = 0.0
    for k, s in enumerate(seqs):
        want = ref.forward(ref.new_cache(), s, last_only=False)
        slots = [trie.slot_of(k, p) for p in range(len(s))]
        got = torch.cat([lg for _, lg in tor.logits_rows(hid, slots)])
        worst = max(worst, float((got - want).abs().max()))
    # same operations in the same order; only GEMM blocking differs
    assert worst < (1e-4 if exact else 2e-2), worst


def test_summaries():
    row = torch.tensor([0.0, 5.0, 5.0, 1.0] + [-1.0] * 20)
    s = choice_summary(row, 24, 2)
    assert s["argmax"] == 1 and s["margin"] == 0.0 and s["gap"] == 0.0
    row = torch.full((40,), -5.0)
    row[:10] = -20.0
    row[3], row[7] = 2.0, 1.5
    row[20:28] = torch.arange(8, dtype=torch.float32)  # 8 tokens, two of them above both digits
    # both digits are members; the closest decision is digit 3 vs digit 7
    assert readout_ambiguity(row, 40) == pytest.approx(0.5)
