"""Measure the oracle's fp32-vs-fp64 noise floor per model shape at full depth
(the basis of every parity tolerance; committed as tests/golden/floors.json).

For each model: two sequences (a 2K-token generation prompt + CoT, and a
verification prompt over a 1K-word CoT) go through the layer-streamed oracle
(``oracle/tree_oracle.py``) twice -- fp32 and fp64 arithmetic, identical bf16
storage points -- and the floor is max |logits32 - logits64| (and the mean)
over the last 128 positions of each.  The device's own prefill logits of the
same positions are compared with the fp32 oracle for information.

    python tools/measure_floors.py --models r1-1.5b,qwen2.5-7b,qwq-32b --out gpurun_out/floors.json
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from oracle.tree_oracle import PrefixTrie, TreeOracle  # noqa: E402
from paper_2504_07891_b200.backend import B200Backend  # noqa: E402
from paper_2504_07891_b200.domain import (BackendRole, render_generation_prompt,  # noqa: E402
                                          render_verification_prompt)
from paper_2504_07891_b200.shapes import get_spec  # noqa: E402

TAIL = 128


def sequences(vocab, n_gen: int = 2048, n_cot: int = 1024) -> list[list[int]]:
    words = vocab.problem(64 + n_gen + n_cot + 24, 77).split()
    gen = vocab.encode(render_generation_prompt(" ".join(words[:64]), " ".join(words[64:64 + n_gen]) + " "))
    ver = vocab.encode(render_verification_prompt(" ".join(words[:64]),
                                                  " ".join(words[64:64 + n_cot]) + " ",
                                                  " ".join(words[-24:]) + " "))
    return [gen, ver]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="tiny-draft,tiny-base,r1-1.5b,qwen2.5-7b,qwq-32b")
    ap.add_argument("--out", default="gpurun_out/floors.json")
    args = ap.parse_args()
    out = {}
    for name in args.models.split(","):
        t0 = time.time()
        spec = get_spec(name)
        be = B200Backend(spec, BackendRole.BASE if spec.judge else BackendRole.SMALL,
                         max_ctx=4096, n_streams=1)
        w = be.device_model.weights
        seqs = sequences(be.vocab)
        res = {}
        for dt in (torch.float32, torch.float64):
            trie = PrefixTrie()
            for s in seqs:
                trie.insert(s)
            orc = TreeOracle(spec, lambda n: w[n], device="cuda", dtype=dt)
            hid = orc.hidden(trie)
            rows = []
            for k, s in enumerate(seqs):
                sl = trie.slots_of(k, list(range(len(s) - TAIL, len(s))))
                rows.append(torch.cat([r for _, r in orc.logits_rows(hid, sl)])[:, : spec.vocab_text])
            res[dt] = torch.cat(rows).double()
            del hid
        d = (res[torch.float32] - res[torch.float64]).abs()
        # the device's prefill logits of the same positions (information only)
        eng, st = be.engine, be.pool.streams[0]
        dev_err = []
        for k, s in enumerate(seqs):
            eng.truncate(st, 0)
            eng.prefill(st, s[:-TAIL])
            got = eng.forward_logits(st, s[-TAIL:])[:, : spec.vocab_text].double()
            ref = res[torch.float32][k * TAIL:(k + 1) * TAIL].to(got.device)
            dev_err.append((got - ref).abs())
        de = torch.cat(dev_err)
        out[name] = {"floor_max_abs": float(d.max()), "floor_mean_abs": float(d.mean()),
                     "device_max_abs": float(de.max()), "device_mean_abs": float(de.mean()),
                     "positions": 2 * TAIL, "contexts": [len(s) for s in seqs],
                     "layers": spec.n_layers, "seconds": round(time.time() - t0, 1)}
        print(json.dumps({name: out[name]}), flush=True)
        del be, res
        torch.cuda.empty_cache()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
