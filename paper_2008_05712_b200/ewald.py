"""Ewald kernel class.

The reference's NBodyWorkload can submit a second kernel class, "ewald": one
work request per bucket with buffers [bucket] and item_count max(1, n_b)
(hr/workloads/nbody.py:317-323); the simulator only charges its modelled cost
(hr/devicesim.py:92-99, KERNEL_PRESETS "ewald").  On the B200 the class
computes what a ChaNGa-style periodic code needs from it: the Ewald
correction of every particle from the root multipole (monopole + traceless
quadrupole), float64, in csrc/ewald.cuh.  With the correction, the periodic
force of particle i is the tree force plus ``g m_i a_corr``.

There is no reference arithmetic for this class ("parity unpinned"); the
float64 oracle (oracle/gcharm_oracle.c orc_ewald_correction) is pinned by
known answers in tests/test_ewald_cpu.py and the device path is checked
against it in tests/test_ewald_gpu.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass(frozen=True)
class EwaldParams:
    """Box side, real/Fourier split and cut-offs (ChaNGa defaults: alpha =
    2 / L, real-space replicas |n_k| <= 3 within 2.6 L, |m| <= 2.8)."""
    L: float = 1.0
    alpha: float | None = None
    nrep: int = 3
    ewcut: float = 2.6
    hcut: float = 2.8

    def array(self) -> np.ndarray:
        a = 2.0 / self.L if self.alpha is None else self.alpha
        return np.array([self.L, a, self.nrep, self.ewcut, self.hcut], float)


def multipole_moments(pos, mass, ctx=None) -> np.ndarray:
    """[M, com(3), Q xx yy zz xy xz yz] of a 3-D distribution (device reduction)."""
    pos, mass = L.f64(pos), L.f64(mass)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError("Ewald summation needs 3-D positions")
    out = np.zeros(10)
    c = ctx or L.context()
    L.call("gc_ewald_moments", c.handle, len(pos), L.ptr(pos, L.f64p), L.ptr(mass, L.f64p), L.ptr(out, L.f64p))
    return out


def ewald_correction(pos, moments, params: EwaldParams = EwaldParams(), ctx=None):
    """Correction acceleration (n, 3) and potential (n,) at `pos` (G = 1)."""
    pos, mom = L.f64(pos), L.f64(moments)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError("Ewald summation needs 3-D positions")
    n = len(pos)
    acc, pot = np.zeros((n, 3)), np.zeros(n)
    c = ctx or L.context()
    L.call("gc_ewald_correction", c.handle, n, L.ptr(pos, L.f64p), L.ptr(mom, L.f64p),
           L.ptr(params.array(), L.f64p), L.ptr(acc, L.f64p), L.ptr(pot, L.f64p))
    return acc, pot


def tree_moments(tree) -> np.ndarray:
    """Root multipole of a device tree's particles (gc_bh_ewald_moments)."""
    out = np.zeros(10)
    L.call("gc_bh_ewald_moments", tree.handle, L.ptr(out, L.f64p))
    return out
