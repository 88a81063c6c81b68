"""ctypes wrapper over gcharm_oracle.c — CPU ORACLE, test infrastructure only.

Mirrors the reference call signatures so tests read like the reference's:
``build_bucket_tree`` (hr/workloads/nbody.py:78), ``build_interaction_lists``
(nbody.py:160), ``eval_forces`` (nbody.py:216), ``direct_forces``
(hr/kernels.py:40), ``forces_from_points`` (kernels.py:70), ``md_cross_forces`` /
``md_self_forces`` (kernels.py:105-156), ``compute_forces`` (md.py:121) and the
3-D LJ restatement (no reference; parity unpinned).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgcharm_oracle.so")
_lib = None

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
i8p = C.POINTER(C.c_int8)
i32p = C.POINTER(C.c_int32)


class _Tree(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64), ("n_buckets", C.c_int64),
        ("center", f64p), ("half", f64p), ("mass", f64p), ("com", f64p),
        ("first_child", i64p), ("n_child", i32p), ("pstart", i64p), ("pcount", i64p),
        ("buckets", i64p), ("pidx", i64p),
    ]


def build():
    """Compile the oracle (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "gcharm_oracle.c")
        ):
            build()
        L = C.CDLL(_SO)
        L.orc_build_tree.argtypes = [C.c_int64, C.c_int, f64p, f64p, C.c_double, C.c_int64, C.POINTER(_Tree)]
        L.orc_free_tree.argtypes = [C.POINTER(_Tree)]
        L.orc_build_tree_forced.argtypes = [C.c_int64, C.c_int, f64p, f64p, C.c_double, C.c_int64, C.c_int64,
                                            i32p, C.POINTER(C.c_uint64), C.POINTER(_Tree)]
        L.orc_build_lists.argtypes = [C.POINTER(_Tree), C.c_int, C.c_double, i64p,
                                      C.POINTER(i64p), C.POINTER(i8p), i64p, C.c_int]
        L.orc_build_lists_range.argtypes = [C.POINTER(_Tree), C.c_int, C.c_double, C.c_int64, C.c_int64, i64p,
                                            C.POINTER(i64p), C.POINTER(i8p), i64p, C.c_int]
        L.orc_eval_forces.argtypes = [C.POINTER(_Tree), C.c_int, f64p, f64p, i64p, i64p, i8p,
                                      C.c_int64, C.c_int64, C.c_double, C.c_double, f64p, C.c_int]
        L.orc_eval_potentials.argtypes = L.orc_eval_forces.argtypes
        L.orc_periodic_forces.argtypes = [C.POINTER(_Tree), C.c_int, C.c_double, C.c_double, C.c_int, f64p, f64p,
                                          C.c_int64, C.c_int64, C.c_double, C.c_double, f64p, i64p, i64p, C.c_int]
        L.orc_forces_from_points.argtypes = [C.c_int64, C.c_int64, C.c_int, f64p, f64p, f64p, f64p,
                                             C.c_double, C.c_double, f64p]
        L.orc_direct_forces.argtypes = [C.c_int64, C.c_int, f64p, f64p, C.c_double, C.c_double, f64p, C.c_int]
        L.orc_md_cross_forces.argtypes = [C.c_int64, C.c_int64, C.c_int, f64p, f64p, C.c_double,
                                          C.c_double, f64p, f64p]
        L.orc_md_self_forces.argtypes = [C.c_int64, C.c_int, f64p, C.c_double, C.c_double, f64p]
        L.orc_md2d_compute_forces.argtypes = [C.c_int64, f64p, i64p, C.c_int64, C.c_int64, C.c_double,
                                              C.c_double, C.c_double, C.c_int, f64p]
        L.orc_lj3d_compute_forces.argtypes = [C.c_int64, f64p, i64p, C.c_double, C.c_double, C.c_double,
                                              C.c_double, C.c_int, f64p, f64p, C.c_int]
        L.orc_lj3d_bruteforce.argtypes = [C.c_int64, f64p, f64p, C.c_double, C.c_double, C.c_double,
                                          C.c_int, f64p, f64p]
        L.orc_count_address_runs.argtypes = [i64p, C.c_int64, C.c_int64]
        L.orc_count_address_runs.restype = C.c_int64
        L.orc_pairwise_sum.argtypes = [f64p, C.c_int64]
        L.orc_pairwise_sum.restype = C.c_double
        L.orc_num_threads.restype = C.c_int
        L.orc_ewald_moments.argtypes = [C.c_int64, f64p, f64p, f64p]
        L.orc_ewald_correction.argtypes = [C.c_int64, f64p, f64p, C.c_double, C.c_double, C.c_int, C.c_double,
                                           C.c_double, f64p, f64p]
        L.free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


@dataclass
class OracleTree:
    """Flat form of BucketTree (nbody.py:71-75): node ids are level order."""

    dim: int
    center: np.ndarray  # (n_nodes, dim)
    half: np.ndarray
    mass: np.ndarray
    com: np.ndarray  # (n_nodes, dim)
    first_child: np.ndarray  # -1 for buckets
    n_child: np.ndarray
    pstart: np.ndarray
    pcount: np.ndarray
    buckets: np.ndarray  # DFS order
    pidx: np.ndarray

    @property
    def n_nodes(self):
        return len(self.half)

    def particle_idx(self, node):
        return self.pidx[self.pstart[node]: self.pstart[node] + self.pcount[node]]

    def _ctree(self):
        t = _Tree()
        t.n_nodes = self.n_nodes
        t.n_buckets = len(self.buckets)
        self._keep = [_f64(self.center).ravel(), _f64(self.half), _f64(self.mass), _f64(self.com).ravel(),
                      np.ascontiguousarray(self.first_child, np.int64), np.ascontiguousarray(self.n_child, np.int32),
                      np.ascontiguousarray(self.pstart, np.int64), np.ascontiguousarray(self.pcount, np.int64),
                      np.ascontiguousarray(self.buckets, np.int64), np.ascontiguousarray(self.pidx, np.int64)]
        k = self._keep
        t.center, t.half, t.mass, t.com = _p(k[0], f64p), _p(k[1], f64p), _p(k[2], f64p), _p(k[3], f64p)
        t.first_child, t.n_child, t.pstart, t.pcount = _p(k[4], i64p), _p(k[5], i32p), _p(k[6], i64p), _p(k[7], i64p)
        t.buckets, t.pidx = _p(k[8], i64p), _p(k[9], i64p)
        return t


@dataclass
class OracleLists:
    """CSR of InteractionList (nbody.py:146-152) over buckets in DFS order."""

    ptr: np.ndarray  # (n_buckets+1,)
    ids: np.ndarray  # walk_order node ids
    kind: np.ndarray  # 0 = node_interactions, 1 = particle_interactions
    item_count: np.ndarray

    def walk_order(self, b):
        return self.ids[self.ptr[b]: self.ptr[b + 1]]

    def node_interactions(self, b):
        s = slice(self.ptr[b], self.ptr[b + 1])
        return self.ids[s][self.kind[s] == 0]

    def particle_interactions(self, b):
        s = slice(self.ptr[b], self.ptr[b + 1])
        return self.ids[s][self.kind[s] == 1]


def octant_keys(positions, box=1.0):
    """Restatement of the device build's octant keys (bh_build.cu bb_keys =
    the descent of hr/workloads/nbody.py:97-108): level L digit
    q = sum_k (x_k >= c_k) << k at bits 3 (20 - L) of k1 (L < 21) or
    3 (41 - L) of k2; levels with half < 1e-9 contribute nothing."""
    pos = _f64(positions)
    n, dim = pos.shape
    nlev, h = 0, box / 2.0
    while h >= 1e-9 and nlev <= 42:
        nlev += 1
        h /= 2.0
    c = np.full((n, dim), box * 0.5)
    h = box * 0.5
    k1 = np.zeros(n, np.uint64)
    k2 = np.zeros(n, np.uint64)
    for L in range(nlev):
        q = np.zeros(n, np.uint64)
        for k in range(dim):
            q |= (pos[:, k] >= c[:, k]).astype(np.uint64) << np.uint64(k)
        if L < 21:
            k1 |= q << np.uint64(3 * (20 - L))
        else:
            k2 |= q << np.uint64(3 * (41 - L))
        ch = h * 0.5
        for k in range(dim):
            c[:, k] = c[:, k] + np.where((q >> np.uint64(k)) & np.uint64(1), ch, -ch)
        h = ch
    return k1, k2


def build_bucket_tree(positions, masses, bucket_size, box=1.0, forced=None) -> OracleTree:
    """forced=(levels int32 (m,), prefixes uint64 (m, 2)): cubes split whatever
    their count (the distributed build's straddling cubes)."""
    L = lib()
    pos = _f64(positions)
    n, dim = pos.shape
    m = _f64(masses)
    t = _Tree()
    if forced is not None and len(forced[0]):
        fl = np.ascontiguousarray(forced[0], np.int32)
        fp = np.ascontiguousarray(forced[1], np.uint64).reshape(-1)
        rc = L.orc_build_tree_forced(n, dim, _p(pos, f64p), _p(m, f64p), float(box), int(bucket_size), len(fl),
                                     _p(fl, i32p), fp.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(t))
    else:
        rc = L.orc_build_tree(n, dim, _p(pos, f64p), _p(m, f64p), float(box), int(bucket_size), C.byref(t))
    if rc != 0:
        raise ValueError(f"orc_build_tree failed ({rc})")
    nn = t.n_nodes
    out = OracleTree(
        dim=dim,
        center=_copy(t.center, nn * dim, np.float64).reshape(nn, dim),
        half=_copy(t.half, nn, np.float64),
        mass=_copy(t.mass, nn, np.float64),
        com=_copy(t.com, nn * dim, np.float64).reshape(nn, dim),
        first_child=_copy(t.first_child, nn, np.int64),
        n_child=_copy(t.n_child, nn, np.int32),
        pstart=_copy(t.pstart, nn, np.int64),
        pcount=_copy(t.pcount, nn, np.int64),
        buckets=_copy(t.buckets, t.n_buckets, np.int64),
        pidx=_copy(t.pidx, n, np.int64),
    )
    L.orc_free_tree(C.byref(t))
    return out


def build_interaction_lists(tree: OracleTree, theta, nthreads=0, bucket_range=None) -> OracleLists:
    """bucket_range=(b0, b1): walk only those DFS buckets (the rest get empty lists)."""
    L = lib()
    ct = tree._ctree()
    nb = len(tree.buckets)
    ptr = np.zeros(nb + 1, np.int64)
    ic = np.zeros(nb, np.int64)
    ids_p, kind_p = i64p(), i8p()
    b0, b1 = (0, nb) if bucket_range is None else bucket_range
    rc = L.orc_build_lists_range(C.byref(ct), tree.dim, float(theta), int(b0), int(b1), _p(ptr, i64p),
                                 C.byref(ids_p), C.byref(kind_p), _p(ic, i64p), int(nthreads))
    if rc != 0:
        raise ValueError("theta must be >= 0")
    tot = int(ptr[-1])
    ids = _copy(ids_p, tot, np.int64)
    kind = _copy(kind_p, tot, np.int8)
    L.free(C.cast(ids_p, C.c_void_p))
    L.free(C.cast(kind_p, C.c_void_p))
    return OracleLists(ptr=ptr, ids=ids, kind=kind, item_count=ic)


def eval_forces(tree: OracleTree, lists: OracleLists, positions, masses, g=1.0, eps=1e-4,
                bucket_range=None, nthreads=0):
    L = lib()
    ct = tree._ctree()
    pos, m = _f64(positions), _f64(masses)
    n = pos.shape[0]
    out = np.zeros((n, tree.dim))
    b0, b1 = (0, len(tree.buckets)) if bucket_range is None else bucket_range
    ptr = np.ascontiguousarray(lists.ptr, np.int64)
    ids = np.ascontiguousarray(lists.ids, np.int64)
    kind = np.ascontiguousarray(lists.kind, np.int8)
    L.orc_eval_forces(C.byref(ct), tree.dim, _p(pos, f64p), _p(m, f64p), _p(ptr, i64p), _p(ids, i64p),
                      _p(kind, i8p), int(b0), int(b1), float(g), float(eps), _p(out, f64p), int(nthreads))
    return out


def periodic_forces(tree: OracleTree, positions, masses, theta, L=1.0, nrep=1, g=1.0, eps=1e-4,
                    bucket_range=None, nthreads=0):
    """Periodic BH restatement (no reference implementation: parity
    unpinned): every bucket walks the tree once per image shift of the box
    (side L, (2 nrep + 1)^3 images) with shifted centres of mass in the
    opening test; returns (forces, entries per bucket, items per bucket)."""
    lb = lib()
    ct = tree._ctree()
    pos, m = _f64(positions), _f64(masses)
    n = pos.shape[0]
    out = np.zeros((n, 3))
    nb = len(tree.buckets)
    b0, b1 = (0, nb) if bucket_range is None else bucket_range
    ent = np.zeros(nb, np.int64)
    itm = np.zeros(nb, np.int64)
    rc = lb.orc_periodic_forces(C.byref(ct), tree.dim, float(theta), float(L), int(nrep), _p(pos, f64p), _p(m, f64p),
                                int(b0), int(b1), float(g), float(eps), _p(out, f64p), _p(ent, i64p), _p(itm, i64p),
                                int(nthreads))
    if rc != 0:
        raise ValueError("orc_periodic_forces: bad arguments (3-D, 0 <= nrep <= 2)")
    return out, ent, itm


def eval_potentials(tree: OracleTree, lists: OracleLists, positions, masses, g=1.0, eps=1e-4,
                    bucket_range=None, nthreads=0):
    """Per-particle potential -g m_i sum_j m_j / sqrt(r^2 + eps^2) over the
    interaction lists (restated beside forces_from_points, hr/kernels.py:70-88;
    no reference counterpart: parity unpinned, pinned by the direct sum at
    theta = 0 in tests/test_oracle_golden.py)."""
    L = lib()
    ct = tree._ctree()
    pos, m = _f64(positions), _f64(masses)
    out = np.zeros(pos.shape[0])
    b0, b1 = (0, len(tree.buckets)) if bucket_range is None else bucket_range
    ptr = np.ascontiguousarray(lists.ptr, np.int64)
    ids = np.ascontiguousarray(lists.ids, np.int64)
    kind = np.ascontiguousarray(lists.kind, np.int8)
    L.orc_eval_potentials(C.byref(ct), tree.dim, _p(pos, f64p), _p(m, f64p), _p(ptr, i64p), _p(ids, i64p),
                          _p(kind, i8p), int(b0), int(b1), float(g), float(eps), _p(out, f64p), int(nthreads))
    return out


def direct_forces(pos, mass, g=1.0, eps=1e-4, nthreads=0):
    pos, mass = _f64(pos), _f64(mass)
    n, dim = pos.shape
    out = np.zeros((n, dim))
    lib().orc_direct_forces(n, dim, _p(pos, f64p), _p(mass, f64p), float(g), float(eps), _p(out, f64p),
                            int(nthreads))
    return out


def forces_from_points(ppos, pmass, spos, smass, g, eps):
    ppos, pmass, spos, smass = _f64(ppos), _f64(pmass), _f64(spos), _f64(smass)
    n, dim = ppos.shape
    out = np.zeros((n, dim))
    lib().orc_forces_from_points(n, spos.shape[0], dim, _p(ppos, f64p), _p(pmass, f64p), _p(spos, f64p),
                                 _p(smass, f64p), float(g), float(eps), _p(out, f64p))
    return out


def md_cross_forces(pa, pb, cutoff, stiffness):
    pa, pb = _f64(pa), _f64(pb)
    fa, fb = np.zeros_like(pa), np.zeros_like(pb)
    lib().orc_md_cross_forces(pa.shape[0], pb.shape[0], pa.shape[1], _p(pa, f64p), _p(pb, f64p),
                              float(cutoff), float(stiffness), _p(fa, f64p), _p(fb, f64p))
    return fa, fb


def md_self_forces(p, cutoff, stiffness):
    p = _f64(p)
    out = np.zeros_like(p)
    lib().orc_md_self_forces(p.shape[0], p.shape[1], _p(p, f64p), float(cutoff), float(stiffness), _p(out, f64p))
    return out


def md2d_compute_forces(positions, patch_of, rows, cols, patch_size, cutoff, stiffness=25.0, periodic=False):
    pos = _f64(positions)
    po = np.ascontiguousarray(patch_of, np.int64)
    out = np.zeros_like(pos)
    lib().orc_md2d_compute_forces(pos.shape[0], _p(pos, f64p), _p(po, i64p), int(rows), int(cols),
                                  float(patch_size), float(cutoff), float(stiffness), int(bool(periodic)),
                                  _p(out, f64p))
    return out


def md2d_step(positions, velocities, patch_of, rows, cols, patch_size, cutoff, dt, stiffness=25.0,
              periodic=False):
    """md_step (md.py:166-190) restated; returns (positions, velocities, patch_of)."""
    forces = md2d_compute_forces(positions, patch_of, rows, cols, patch_size, cutoff, stiffness, periodic)
    vel = velocities + forces * dt
    pos = positions + vel * dt
    hi = np.array([rows * patch_size, cols * patch_size])
    if periodic:
        pos = pos % hi
    else:
        for k in range(2):
            below = pos[:, k] < 0.0
            pos[below, k] = -pos[below, k]
            vel[below, k] *= -1.0
            above = pos[:, k] > hi[k]
            pos[above, k] = 2.0 * hi[k] - pos[above, k]
            vel[above, k] *= -1.0
        pos = np.clip(pos, 0.0, hi - 1e-12)
    r = np.minimum((pos[:, 0] // patch_size).astype(np.int64), rows - 1)
    c = np.minimum((pos[:, 1] // patch_size).astype(np.int64), cols - 1)
    return pos, vel, r * cols + c


def lj3d_compute_forces(positions, dims, cell_size, rc=2.5, eps=1.0, sigma=1.0, periodic=True, nthreads=1):
    """nthreads=1: the serial parity restatement; otherwise (0 = all) the
    multi-core form used as the CPU baseline (same pairs, thread-private sums)."""
    pos = _f64(positions)
    d = np.ascontiguousarray(dims, np.int64)
    f = np.zeros_like(pos)
    e = np.zeros(pos.shape[0])
    lib().orc_lj3d_compute_forces(pos.shape[0], _p(pos, f64p), _p(d, i64p), float(cell_size), float(rc),
                                  float(eps), float(sigma), int(bool(periodic)), _p(f, f64p), _p(e, f64p),
                                  int(nthreads))
    return f, e


def lj3d_bruteforce(positions, box, rc=2.5, eps=1.0, sigma=1.0, periodic=True):
    pos = _f64(positions)
    b = _f64(box)
    f = np.zeros_like(pos)
    e = np.zeros(pos.shape[0])
    lib().orc_lj3d_bruteforce(pos.shape[0], _p(pos, f64p), _p(b, f64p), float(rc), float(eps), float(sigma),
                              int(bool(periodic)), _p(f, f64p), _p(e, f64p))
    return f, e


def lj3d_step(positions, velocities, dims, cell_size, dt, rc=2.5, eps=1.0, sigma=1.0, nthreads=1):
    """LJ analogue of md_step (md.py:166-190) with periodic wrap: v += F dt
    (unit mass); x += v dt; x %= box.  Returns (pos, vel, forces, energy)."""
    f, e = lj3d_compute_forces(positions, dims, cell_size, rc, eps, sigma, True, nthreads)
    vel = velocities + f * dt
    pos = positions + vel * dt
    box = np.asarray(dims, np.float64) * cell_size
    pos = pos % box
    return pos, vel, f, e


def ewald_moments(pos, mass):
    """Root multipole of a 3-D distribution: [M, com(3), traceless Q (xx, yy, zz, xy, xz, yz)]."""
    pos, mass = _f64(pos), _f64(mass)
    out = np.zeros(10)
    lib().orc_ewald_moments(pos.shape[0], _p(pos, f64p), _p(mass, f64p), _p(out, f64p))
    return out


def ewald_correction(pos, moments, L=1.0, alpha=None, nrep=3, ewcut=2.6, hcut=2.8):
    """Periodic (Ewald) correction acceleration + potential at `pos` from the
    multipole `moments` (restatement in gcharm_oracle.c; parity unpinned --
    the reference only models the ewald class)."""
    pos, mom = _f64(pos), _f64(moments)
    n = pos.shape[0]
    acc, pot = np.zeros((n, 3)), np.zeros(n)
    alpha = 2.0 / L if alpha is None else alpha
    lib().orc_ewald_correction(n, _p(pos, f64p), _p(mom, f64p), float(L), float(alpha), int(nrep), float(ewcut),
                               float(hcut), _p(acc, f64p), _p(pot, f64p))
    return acc, pot


def count_address_runs(addresses, group=16):
    a = np.ascontiguousarray(addresses, np.int64)
    return int(lib().orc_count_address_runs(_p(a, i64p), a.shape[0], int(group)))


def pairwise_sum(a):
    a = _f64(a)
    return float(lib().orc_pairwise_sum(_p(a, f64p), a.shape[0]))


def num_threads():
    return int(lib().orc_num_threads())
