"""Bring-up probe: decode a few tokens on each named model under a watchdog;
on a hang, print the persistent kernel's per-CTA progress words (SR_MK_TRACE)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SR_MK_TRACE", "1")
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2504_07891_b200 import native  # noqa: E402
from paper_2504_07891_b200.backend import B200Backend  # noqa: E402
from paper_2504_07891_b200.domain import BackendRole  # noqa: E402
from paper_2504_07891_b200.shapes import get_spec  # noqa: E402

for name in sys.argv[1:]:
    spec = get_spec(name)
    b = B200Backend(spec, BackendRole.SMALL, max_ctx=1024)
    ids = list(range(16, 100))
    res = {}

    def run():
        res["out"] = b.engine.generate(b.pool.streams[0], ids, 8, ())

    th = threading.Thread(target=run, daemon=True)
    t = time.time()
    th.start()
    th.join(20)
    if th.is_alive():
        n = torch.cuda.get_device_properties(0).multi_processor_count
        buf = (C.c_int32 * (n * 8))()
        native.load().sr_debug_trace(b.device_model.handle, buf, n * 8)
        rows = [list(buf[i * 8:i * 8 + 5]) for i in range(n)]
        print(name, "HANG; per-CTA [step, consumed, target, issued, n_gen]:", flush=True)
        for i, r in enumerate(rows):
            print(i, r, flush=True)
        os._exit(3)
    print(name, "ok", res.get("out"), round(time.time() - t, 3), flush=True)
