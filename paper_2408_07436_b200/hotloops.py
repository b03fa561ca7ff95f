"""Kernel-level drop-in for the reference ``kifmm3d.hotloops`` module
(``hotloops.py:13-77``): same function names, argument order and
accumulate/overwrite semantics, with host numpy arrays in and out, but
every loop runs on the GPU through ``libkifmm_b200.so``.

``BACKEND`` is ``"cuda"``; there is no compiled-CPU or NumPy fallback (the
reference's ``KIFMM_PURE_PYTHON`` switch has no counterpart).  ``threads``
arguments are accepted and ignored.
"""

from __future__ import annotations

import numpy as np

BACKEND = "cuda"
COMPILED = True


def resolve_threads(threads=None) -> int:
    from .engine import _resolve_threads
    return _resolve_threads(threads)


def _check_dtype(*arrays):
    dt = np.asarray(arrays[0]).dtype
    if dt not in (np.float32, np.float64):
        raise TypeError(f"unsupported dtype {dt}")
    for a in arrays[1:]:
        if np.asarray(a).dtype != dt:
            raise ValueError("all real arrays must share one dtype")
    return dt


def _upload(*arrays, dtype=None):
    """Device copies, returned as a list the caller keeps alive for the
    duration of the launch (raw pointers do not hold a reference)."""
    from .device import to_dev
    return [to_dev(a, dtype) for a in arrays]


def _sfx(dt):
    return "f32" if dt == np.float32 else "f64"


def laplace_potentials(tx, ty, tz, sx, sy, sz, charges, out, threads=None):
    """out[i, r] += sum_j K(t_i, s_j) q[j, r]  (reference _hot.pyx:24-65)."""
    from . import _native as nat
    from .device import P, require_cuda, stream_handle
    require_cuda()
    dt = _check_dtype(tx, ty, tz, sx, sy, sz, charges, out)
    nt, ns = np.asarray(tx).shape[0], np.asarray(sx).shape[0]
    q = np.ascontiguousarray(charges).reshape(ns, -1)
    d = _upload(tx, ty, tz, sx, sy, sz, q, np.ascontiguousarray(out).reshape(nt, -1))
    if nt and ns:
        nat.call(f"kifmm_laplace_potentials_{_sfx(dt)}", P(d[0]), P(d[1]), P(d[2]), nt, P(d[3]),
                 P(d[4]), P(d[5]), ns, P(d[6]), q.shape[1], P(d[7]), stream_handle())
    out[...] = d[7].cpu().numpy().reshape(np.shape(out))
    return out


def laplace_gradients(tx, ty, tz, sx, sy, sz, charges, out, grad, threads=None):
    """out[i, r] += sum_j K q, grad[i, r, :] += sum_j q grad_t K (extension of
    laplace_potentials; the reference has no gradient loop).  ``grad`` is
    shaped ``out.shape + (3,)``."""
    from . import _native as nat
    from .device import P, require_cuda, stream_handle
    require_cuda()
    dt = _check_dtype(tx, ty, tz, sx, sy, sz, charges, out, grad)
    nt, ns = np.asarray(tx).shape[0], np.asarray(sx).shape[0]
    q = np.ascontiguousarray(charges).reshape(ns, -1)
    if np.shape(grad) != tuple(np.shape(out)) + (3,):
        raise ValueError("grad must be shaped out.shape + (3,)")
    d = _upload(tx, ty, tz, sx, sy, sz, q, np.ascontiguousarray(out).reshape(nt, -1),
                np.ascontiguousarray(grad).reshape(nt, -1))
    if nt and ns:
        nat.call(f"kifmm_laplace_gradients_{_sfx(dt)}", P(d[0]), P(d[1]), P(d[2]), nt, P(d[3]),
                 P(d[4]), P(d[5]), ns, P(d[6]), q.shape[1], P(d[7]), P(d[8]), stream_handle())
    out[...] = d[7].cpu().numpy().reshape(np.shape(out))
    grad[...] = d[8].cpu().numpy().reshape(np.shape(grad))
    return out, grad


def laplace_matrix(tx, ty, tz, sx, sy, sz, out=None, threads=None):
    """out[i, j] = K(t_i, s_j), overwritten (reference _hot.pyx:68-88)."""
    import torch

    from . import _native as nat
    from .device import P, require_cuda, stream_handle
    require_cuda()
    dt = _check_dtype(tx, ty, tz, sx, sy, sz)
    nt, ns = np.asarray(tx).shape[0], np.asarray(sx).shape[0]
    if out is None:
        out = np.empty((nt, ns), dtype=dt)
    d = _upload(tx, ty, tz, sx, sy, sz)
    o = torch.empty(max(nt * ns, 1), dtype=torch.float32 if dt == np.float32 else torch.float64,
                    device=d[0].device)
    if nt and ns:
        nat.call(f"kifmm_laplace_matrix_{_sfx(dt)}", P(d[0]), P(d[1]), P(d[2]), nt, P(d[3]),
                 P(d[4]), P(d[5]), ns, P(o), stream_handle())
        out[...] = o[: nt * ns].cpu().numpy().reshape(nt, ns)
    return out


def p2p_blocked(tx, ty, tz, leaf_of_target, sx, sy, sz, charges, src_offsets, out, threads=None):
    """Near-field sweep over the gathered CSR (reference _hot.pyx:91-138)."""
    from . import _native as nat
    from .device import P, require_cuda, stream_handle
    require_cuda()
    dt = _check_dtype(tx, ty, tz, sx, sy, sz, charges, out)
    nt = np.asarray(tx).shape[0]
    ns = np.asarray(sx).shape[0]
    q = np.ascontiguousarray(charges).reshape(ns, -1)
    d = _upload(tx, ty, tz, sx, sy, sz, q, np.ascontiguousarray(out).reshape(nt, -1))
    idx = _upload(leaf_of_target, src_offsets, dtype=np.int64)
    n_leaves = np.asarray(src_offsets).shape[0] - 1
    if nt:
        nat.call(f"kifmm_p2p_blocked_{_sfx(dt)}", P(d[0]), P(d[1]), P(d[2]), nt, P(idx[0]),
                 P(d[3]), P(d[4]), P(d[5]), P(d[6]), q.shape[1], P(idx[1]), n_leaves, P(d[7]),
                 stream_handle())
    out[...] = d[7].cpu().numpy().reshape(np.shape(out))
    return out


def hadamard_m2l(khat, qhat, halo, phat, block=32, threads=None):
    """phat += frequency-major halo block MAC (reference _hot.pyx:141-178)."""
    from . import _native as nat
    from .device import P, require_cuda, stream_handle
    require_cuda()
    k_, q_, p_ = (np.asarray(a) for a in (khat, qhat, phat))
    if k_.dtype not in (np.complex64, np.complex128):
        raise TypeError(f"unsupported dtype {k_.dtype}")
    if q_.dtype != k_.dtype or p_.dtype != k_.dtype:
        raise ValueError("khat, qhat and phat must share one complex dtype")
    rdt = np.float32 if k_.dtype == np.complex64 else np.float64
    nf, nsc, _, nrhs = q_.shape
    ntc = np.asarray(halo).shape[0]
    d = _upload(*(np.ascontiguousarray(a).view(rdt) for a in (k_, q_, p_)))
    h = _upload(halo, dtype=np.int64)
    nat.call("kifmm_hadamard_m2l_" + ("c64" if rdt == np.float32 else "c128"), P(d[0]), P(d[1]),
             P(h[0]), P(d[2]), nf, nsc, ntc, nrhs, stream_handle())
    phat[...] = d[2].cpu().numpy().view(k_.dtype).reshape(p_.shape)
    return phat
