"""Bring-up aid: two tensor-parallel ranks of the tiny base sharing one GPU
(threads + streams, peer transport), token ids per rank vs the unsharded
model, for growing max_new (1 = host-driven first choice only)."""
import os
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SR_MK_CTAS"] = os.environ.get("SR_MK_CTAS", "72")
import torch  # noqa: E402

from paper_2504_07891_b200.backend import B200Backend, TensorParallel  # noqa: E402
from paper_2504_07891_b200.domain import BackendRole, render_generation_prompt  # noqa: E402
from paper_2504_07891_b200.shapes import get_spec, make_weights  # noqa: E402
from paper_2504_07891_b200.vocab import shared_vocab  # noqa: E402


def on_ranks(bes, fn):
    out = [None] * len(bes)
    err = []

    def work(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(bes[r])
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            err.append(repr(e))

    ts = [threading.Thread(target=work, args=(r,)) for r in range(len(bes))]
    [t.start() for t in ts]
    [t.join(60) for t in ts]
    return out, err, [t.is_alive() for t in ts]


spec = get_spec(sys.argv[1] if len(sys.argv) > 1 else "tiny-base")
w = make_weights(spec, 0)
v = shared_vocab(spec.vocab_text)
full = B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024)
tps = TensorParallel.local_group(2)
ranks = [B200Backend(spec, BackendRole.BASE, weights=w, max_ctx=1024, tp=tps[r]) for r in range(2)]
ids = v.encode(render_generation_prompt(v.problem(64, 30), ""))
# prefill logits: sum of the rank shards' vocab slices vs the full model
def fl(be):
    st = be.pool.streams[1]
    be.engine.truncate(st, 0)
    return be.engine.forward_logits(st, ids).float().cpu()
import time as _t
_t0 = _t.time()
out, err, alive = on_ranks(ranks, fl)
print(f'rank prefill {_t.time()-_t0:.1f}s err={[e[:160] for e in err]} alive={alive}', flush=True)
ref = fl(full)
if out[0] is not None and out[1] is not None:
    cat = torch.cat([out[0], out[1]], dim=1)[:, : spec.vocab_text]
    print("prefill logits max-abs", float((cat - ref[:, : spec.vocab_text]).abs().max()), err)
else:
    print("prefill err", err, alive)

s = full.pool.streams[0]
full.engine.truncate(s, 0)
want, _ = full.engine.generate(s, ids, 24, ())
print("full   ", want, flush=True)
import time
for n in [int(x) for x in os.environ.get('TP_NS', '1,2,3,8,24').split(',')]:
    t0 = time.time()
    def gen(be, n=n):
        st = be.pool.streams[0]
        be.engine.truncate(st, 0)
        return be.engine.generate(st, ids, n, ())[0]
    out, err, alive = on_ranks(ranks, gen)
    print(f"n={n:2d} ({time.time()-t0:.1f}s) r0", out[0], flush=True)
    print(f"     r1", out[1], err, alive, flush=True)
