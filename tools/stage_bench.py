"""Host->device copy of 8 MB of pageable float64 charges: variants (GPU)."""
import time
from concurrent.futures import ThreadPoolExecutor
import numpy as np
import torch

n = 1_000_000
src_np = np.random.default_rng(0).random(n)
dst = torch.empty(n, dtype=torch.float64, device="cuda")
stage = torch.empty(n, dtype=torch.float64, pin_memory=True)
stage_np = stage.numpy()
pool = ThreadPoolExecutor(8)


def t(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


def direct():
    dst.copy_(torch.from_numpy(src_np))


def pinned_only():
    dst.copy_(stage, non_blocking=True)


def chunked(threads, chunk, use_torch):
    src_t = torch.from_numpy(src_np)
    bounds = [(i, min(n, i + chunk)) for i in range(0, n, chunk)]

    def copy(lo, hi):
        if use_torch:
            stage[lo:hi].copy_(src_t[lo:hi])
        else:
            np.copyto(stage_np[lo:hi], src_np[lo:hi])
    futs = [pool.submit(copy, lo, hi) for lo, hi in bounds]
    for (lo, hi), f in zip(bounds, futs):
        f.result()
        dst[lo:hi].copy_(stage[lo:hi], non_blocking=True)


def whole_torch():
    stage.copy_(torch.from_numpy(src_np))
    dst.copy_(stage, non_blocking=True)


print("torch threads", torch.get_num_threads())
print(f"pageable direct copy_          {t(direct):.3f} ms")
print(f"pinned H2D only                {t(pinned_only):.3f} ms")
print(f"whole torch memcpy + H2D       {t(whole_torch):.3f} ms")
for th in (2, 4, 8):
    for ch in (1 << 16, 1 << 17, 1 << 18):
        for ut in (False, True):
            pool = ThreadPoolExecutor(th)
            print(f"chunked th={th} chunk={ch} torch={ut}  {t(lambda: chunked(th, ch, ut)):.3f} ms")
