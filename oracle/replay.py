"""Teacher-forced replay of a device trajectory through the oracle -- TEST
INFRASTRUCTURE ONLY.

A ``ModelBackend`` constructed with ``record=True`` logs every call it served
(prompt ids, generated ids and the device's top-2 margins, or the judge
readout).  ``replay`` feeds exactly those sequences to the layer-streamed
oracle (``tree_oracle.TreeOracle``) and checks, position by position:

* generation (``Backend.generate_step``, semantics of ``http.py:121-152``):
  each device token must be the oracle's greedy argmax, unless the oracle's
  gap between its argmax and the device token is below the logit tolerance
  -- a *flagged near-tie* (the north-star's rule); where the tokens agree the
  device's reported top1-top2 margin must match the oracle's within the
  tolerance (a logit-level check of the decode path);
* scoring (``Backend.score_step``, ``http.py:154-174`` + ``extract_score``
  ``base.py:106-126`` + ``decide_acceptance`` ``core.py:91-93``): the device
  score and accept bit must equal the oracle's readout (``ref_engine.
  judge_readout``: the top-10 logprob table handed to ``extract_score``),
  unless the readout's deciding logit gap is below the tolerance (flagged).

Teacher forcing makes every call an independent check, so one flagged
near-tie does not end the comparison: the oracle agrees with the device on
the device's own trajectory everywhere outside the flagged positions, which
is the statement "the oracle reproduces the trajectory's tokens, scores and
accept/reject decisions up to flagged near-ties".
"""

from __future__ import annotations

import time
from typing import Any

import torch

from .ref_engine import judge_readout
from .tree_oracle import PrefixTrie, TreeOracle, choice_summary, readout_ambiguity


def replay(backend: Any, calls: list[dict], tol: float, *, device: str = "cuda",
           dtype: torch.dtype = torch.float32, threshold: int | None = None,
           logits_check: int = 0) -> dict:
    """Check ``calls`` (``backend.calls``) against the oracle; returns a report.

    ``logits_check`` > 0 also compares the device's full fp32 logits of the
    last ``logits_check`` positions of the longest generation sequence
    (``sr_forward_logits``, the prefill path) with the oracle's: max-abs."""
    spec = backend.device_model.spec
    weights = backend.device_model.weights
    vocab = backend.vocab
    thr = backend.threshold if threshold is None else threshold
    n_text = vocab.n_text
    t0 = time.time()
    trie = PrefixTrie()
    wanted = []  # (seq index, position, call index, k)
    for ci, c in enumerate(calls):
        if c["kind"] == "gen":
            p, g = c["prompt_ids"], c["gen_ids"]
            if not g:
                continue
            si = trie.insert(p + g[:-1])
            wanted += [(si, len(p) - 1 + k, ci, k) for k in range(len(g))]
        else:
            si = trie.insert(c["prompt_ids"])
            wanted.append((si, len(c["prompt_ids"]) - 1, ci, -1))
    long_seq = None
    if logits_check:
        gens = [i for i, c in enumerate(calls) if c["kind"] == "gen" and c["gen_ids"]]
        if gens:
            ci = max(gens, key=lambda i: len(calls[i]["prompt_ids"]))
            long_seq = list(calls[ci]["prompt_ids"])
            trie.insert(long_seq)
    oracle = TreeOracle(spec, lambda n: weights[n], device=device, dtype=dtype)
    hid = oracle.hidden(trie)
    t_fwd = time.time() - t0
    slots = []
    by_seq: dict[int, list] = {}
    for w in wanted:
        by_seq.setdefault(w[0], []).append(w)
    order = []
    for si, ws in by_seq.items():
        sl = trie.slots_of(si, [w[1] for w in ws])
        slots += sl
        order += ws
    rep = {"model": spec.name, "tol": tol, "tokens": 0, "token_mismatch_flagged": 0,
           "token_mismatch": [], "margin_err_max": 0.0, "scores": 0, "score_mismatch_flagged": 0,
           "score_mismatch": [], "accept_mismatch": 0, "min_token_gap_flagged": None,
           "trie_positions": trie.n_slots, "calls": len(calls)}
    k0 = 0
    for sl, rows in oracle.logits_rows(hid, slots):
        for j, row in enumerate(rows):
            si, pos, ci, k = order[k0 + j]
            c = calls[ci]
            if k >= 0:
                t = c["gen_ids"][k]
                s = choice_summary(row.float(), n_text, t)
                rep["tokens"] += 1
                if t != s["argmax"]:
                    if s["gap"] < tol:
                        rep["token_mismatch_flagged"] += 1
                    else:
                        rep["token_mismatch"].append({"call": ci, "k": k, "device": t,
                                                      "oracle": s["argmax"], "gap": s["gap"]})
                else:
                    m = c.get("margins") or []
                    if len(m) == len(c["gen_ids"]):
                        rep["margin_err_max"] = max(rep["margin_err_max"], abs(m[k] - s["margin"]))
            else:
                rr = row.float().cpu()
                want = judge_readout(rr, vocab, thr)
                amb = readout_ambiguity(rr, n_text)
                rep["scores"] += 1
                if want.score != c["score"]:
                    if amb < tol:
                        rep["score_mismatch_flagged"] += 1
                    else:
                        rep["score_mismatch"].append({"call": ci, "device": c["score"],
                                                      "oracle": want.score, "ambiguity": amb})
                elif bool(want.accept) != bool(c["accept"]):
                    rep["accept_mismatch"] += 1
        k0 += len(sl)
    if long_seq is not None:
        n = min(logits_check, len(long_seq) - 1)
        si = len(trie.seqs) - 1
        sl = trie.slots_of(si, list(range(len(long_seq) - n, len(long_seq))))
        want = torch.cat([r for _, r in oracle.logits_rows(hid, sl)]).float()
        eng = backend.engine
        st = backend.pool.streams[0]
        eng.truncate(st, 0)
        eng.prefill(st, long_seq[:-n])
        got = eng.forward_logits(st, long_seq[-n:]).float()
        eng.truncate(st, 0)
        err = (got[:, :n_text] - want[:, :n_text].to(got.device)).abs().max()
        rep["logits_max_abs"] = float(err)
        rep["logits_rows"] = n
        rep["logits_context"] = len(long_seq)
    rep["oracle_s"] = round(time.time() - t0, 1)
    rep["oracle_forward_s"] = round(t_fwd, 1)
    rep["flagged_rate"] = round((rep["token_mismatch_flagged"] + rep["score_mismatch_flagged"])
                                / max(1, rep["tokens"] + rep["scores"]), 5)
    del hid
    return rep
