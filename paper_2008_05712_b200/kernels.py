"""B200 backend of the reference's kernel module (hr/kernels.py:193-216).

Same function names, argument meaning and float64 results as the reference's
numba/numpy kernels; each call runs one sm_100a kernel through libgcharm.so.
There is no CPU path: without the CUDA library these raise.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L

BACKEND = "cuda-sm_100a"


def _dims(a):
    a = L.f64(a)
    if a.ndim != 2:
        raise ValueError("positions must be (n, dim)")
    return a, a.shape[0], a.shape[1]


def forces_from_points(ppos, pmass, spos, smass, g, eps):
    """hr/kernels.py:70-98: forces on targets from point sources; coincident
    sources are skipped."""
    pp, n, d = _dims(ppos)
    sp, m, d2 = _dims(spos)
    if d2 != d:
        raise ValueError("dimension mismatch")
    pm, sm = L.f64(pmass), L.f64(smass)
    out = np.zeros((n, d))
    L.call("gc_forces_from_points", L.context().handle, n, m, d, L.ptr(pp, L.f64p), L.ptr(pm, L.f64p),
           L.ptr(sp, L.f64p), L.ptr(sm, L.f64p), float(g), float(eps), L.ptr(out, L.f64p))
    return out


def direct_forces(pos, mass, g, eps):
    """hr/kernels.py:40-63: O(n^2) direct summation."""
    p, n, d = _dims(pos)
    m = L.f64(mass)
    out = np.zeros((n, d))
    L.call("gc_direct_forces", L.context().handle, n, d, L.ptr(p, L.f64p), L.ptr(m, L.f64p), float(g),
           float(eps), L.ptr(out, L.f64p))
    return out


def md_cross_forces(pos_a, pos_b, cutoff, stiffness):
    """hr/kernels.py:105-135: soft repulsion between two patches."""
    a, na, d = _dims(pos_a)
    b, nb, _ = _dims(pos_b)
    fa, fb = np.zeros((na, d)), np.zeros((nb, d))
    L.call("gc_md_cross_forces", L.context().handle, na, nb, d, L.ptr(a, L.f64p), L.ptr(b, L.f64p),
           float(cutoff), float(stiffness), L.ptr(fa, L.f64p), L.ptr(fb, L.f64p))
    return fa, fb


def md_self_forces(pos, cutoff, stiffness):
    """hr/kernels.py:138-161: soft repulsion inside one patch."""
    p, n, d = _dims(pos)
    out = np.zeros((n, d))
    L.call("gc_md_self_forces", L.context().handle, n, d, L.ptr(p, L.f64p), float(cutoff), float(stiffness),
           L.ptr(out, L.f64p))
    return out


def count_address_runs(addresses, group: int = 16) -> int:
    """hr/kernels.py:213-216: consecutive-address runs per group-sized chunk."""
    a = L.i64(addresses).ravel()
    out = np.zeros(1, np.int64)
    L.call("gc_count_address_runs", L.context().handle, L.ptr(a, L.i64p), a.shape[0], int(group),
           L.ptr(out, L.i64p))
    return int(out[0])
