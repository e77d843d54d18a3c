"""Logit tolerances of the GPU parity tests, all from the oracle's own noise.

``floor`` = max |oracle fp32 - oracle fp64| logits on identical bf16 storage
points at a model's shape and full depth (``tests/golden/floors.json``,
measured on the B200 by ``tools/measure_floors.py``): how far two exact fp32
implementations of the same bf16-storage model are apart.  The stated
tolerance is ``max(2e-2, 2 * floor)`` -- the north star's example bound, or
twice the floor where the floor is larger.  No tolerance is derived from the
device's own error.
"""

import json
from pathlib import Path

FLOORS = Path(__file__).parent / "golden" / "floors.json"


def floor_tol(model: str) -> float:
    floors = json.loads(FLOORS.read_text())
    return max(2e-2, 2.0 * floors[model]["floor_max_abs"])
