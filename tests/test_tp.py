"""Tensor parallelism of the base model, host side.

* `tp_spec` / `shard_weights` (the sharding the device path loads) partition
  every parameter exactly once;
* the TP decomposition -- row-parallel O and down with an all-reduce after
  each, vocab-parallel LM head with an all-gather -- run on 2 CPU ranks over
  gloo (``oracle/tp_ref.py``) reproduces the unsharded oracle's logits.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_07891_b200.shapes import (gu_split, get_spec, make_weights, shard_weights,
                                          tensor_shapes, tp_spec)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp_spec_divisibility_and_vocab_split():
    spec = get_spec("qwq-32b")
    shards = [tp_spec(spec, r, 8) for r in range(8)]
    assert all(s.n_heads == 5 and s.n_kv_heads == 1 and s.d_ffn == 3456 for s in shards)
    assert sum(s.vocab_rows for s in shards) == spec.vocab_rows
    assert sum(s.vocab_text for s in shards) == spec.vocab_text
    assert [s.vocab_base for s in shards] == [r * 19008 for r in range(8)]
    with pytest.raises(ValueError):
        tp_spec(get_spec("qwen2.5-7b"), 0, 8)  # 4 kv heads do not split 8 ways
    assert tp_spec(spec, 0, 1) is spec


@pytest.mark.parametrize("world", [2])
def test_shards_partition_every_parameter(world):
    spec = get_spec("tiny-base")
    full = make_weights(spec, 0)
    shards = [shard_weights(full, spec, r, world) for r in range(world)]
    for r, sh in enumerate(shards):
        rs = tp_spec(spec, r, world)
        for name, shape in tensor_shapes(rs).items():
            assert tuple(sh[name].shape) == shape, (name, tuple(sh[name].shape), shape)
    # row-parallel / column-parallel pieces reassemble the full tensors
    p = "layers.1."
    assert torch.equal(torch.cat([s[p + "wo"] for s in shards], 1), full[p + "wo"])
    assert torch.equal(torch.cat([s[p + "wd"] for s in shards], 1), full[p + "wd"])
    assert torch.equal(torch.cat([s["lm_head"] for s in shards], 0), full["lm_head"])
    g_full, u_full = gu_split(full[p + "wgu"])
    g = torch.cat([gu_split(s[p + "wgu"])[0] for s in shards])
    u = torch.cat([gu_split(s[p + "wgu"])[1] for s in shards])
    assert torch.equal(g, g_full) and torch.equal(u, u_full)
    hd, qd = spec.head_dim, spec.q_dim
    q = torch.cat([s[p + "wqkv"][: spec.n_heads // world * hd] for s in shards])
    assert torch.equal(q, full[p + "wqkv"][:qd])


def _worker(rank, world, port, ids, out_path):
    from oracle.tp_ref import tp_forward_logits

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    spec = get_spec("tiny-base")
    full = make_weights(spec, 0)
    logits = tp_forward_logits(spec, full, ids, rank, world)
    if rank == 0:
        torch.save(logits, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_decomposition_matches_unsharded_oracle(tmp_path, tiny_vocab):
    from oracle.ref_model import RefModel
    from paper_2504_07891_b200.domain import render_generation_prompt

    spec = get_spec("tiny-base")
    ids = tiny_vocab.encode(render_generation_prompt(tiny_vocab.problem(64, 4), ""))[:48]
    out = tmp_path / "tp_logits.pt"
    mp.spawn(_worker, args=(2, _free_port(), ids, str(out)), nprocs=2, join=True)
    got = torch.load(out)
    ref = RefModel(spec, make_weights(spec, 0))
    want = ref.forward(ref.new_cache(), ids, last_only=False)
    err = (got - want).abs().max().item()
    assert err < 1e-3, err
    # greedy choices agree wherever the oracle is not at a near-tie
    top2 = torch.topk(want[:, : spec.vocab_text], 2).values
    clear = (top2[:, 0] - top2[:, 1]) > 1e-3
    assert torch.equal(got[:, : spec.vocab_text].argmax(-1)[clear],
                       want[:, : spec.vocab_text].argmax(-1)[clear])


def test_make_tp_weights_equals_sliced_full_weights():
    from paper_2504_07891_b200.shapes import make_tp_weights

    spec = get_spec("tiny-base")
    full = make_weights(spec, 0)
    for r in range(2):
        a = make_tp_weights(spec, r, 2, 0)
        b = shard_weights(full, spec, r, 2)
        assert a.keys() == b.keys()
        assert all(torch.equal(a[k], b[k]) for k in a)
