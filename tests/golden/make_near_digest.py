"""Pin the near-field gather plan at BASELINE config-2 size against the
reference's OWN per-leaf loop (engine.py:224-256).

The oracle bridge (oracle/ref_bridge.py) fills the reference instance's
``_near_idx`` / ``_near_offsets`` from our vectorised ``near_field_plan``
because the reference loop takes minutes at 1M points.  This script runs the
unmodified reference ``setup`` once, here (where /root/reference exists), at
config 2 (1M uniform points, seed 7, depth 5) and config 1 (10k, depth 3),
and records SHA-256 digests of the two arrays in near_digest.json;
tests/test_ref_bridge.py::test_near_plan_digest_at_config2_size rebuilds
our plan on the same points and compares.

    python tests/golden/make_near_digest.py        (~6 min)
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import import_reference  # noqa: E402

import_reference()
from kifmm3d import engine  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def main():
    out = {}
    for name, n, depth in (("c1", 10_000, 3), ("c2", 1_000_000, 5)):
        pts = np.random.default_rng(7).random((n, 3))
        cfg = engine.FmmConfig(depth=depth, order_equiv=4, backend="fft", precision="f32")
        t0 = time.perf_counter()
        inst = engine.setup(pts, pts, cfg)
        out[name] = dict(n_points=n, depth=depth, seed=7,
                         near_idx_len=int(inst._near_idx.shape[0]),
                         near_offsets_len=int(inst._near_offsets.shape[0]),
                         n_near_pairs=int(inst.n_near_pairs),
                         near_idx_sha256=digest(inst._near_idx),
                         near_offsets_sha256=digest(inst._near_offsets),
                         reference_setup_seconds=time.perf_counter() - t0)
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "near_digest.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
