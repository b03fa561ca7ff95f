"""Repeated graphed config-2 evaluates (bitwise equal, finite); with an
mbarrier-debug library (tools/build_variant.sh dbg m2l_tmem.cu
-DKIFMM_MBAR_DEBUG) also reports waits that exceeded the debug spin limit."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup, _native
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
fresh_every = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
first = inst.evaluate(q)
bad = 0
for i in range(reps):
    inst2 = setup(pts, pts, FmmConfig(**bench.CONFIG)) if i % fresh_every == fresh_every - 1 \
        else inst
    got = inst2.evaluate(q)
    if not np.array_equal(got, first):
        bad += 1
        d = np.abs(got - first)
        print("mismatch at", i, d.max(), "targets", int((d > 0).sum()),
              "first rows", np.flatnonzero(d > 1e-3 * np.abs(first).max())[:8].tolist())
print("reps", reps, "mismatches", bad, "finite", bool(np.all(np.isfinite(first))))
lib = _native.load()
if hasattr(lib, "kifmm_mbar_debug_read"):
    buf = (ctypes.c_uint * 260)()
    lib.kifmm_mbar_debug_read(buf)
    print("mbar debug stuck waits:", buf[0], [tuple(buf[1 + 4 * k: 5 + 4 * k]) for k in range(min(buf[0], 8))])
