"""Barnes-Hut bucket forces on B200 — the reference's nbody API, device-backed.

Mirrors hr/workloads/nbody.py: ``build_bucket_tree`` (78-120),
``build_interaction_lists`` (160-199), ``eval_forces`` (216-250),
``direct_force_oracle`` (202-213).  The tree lives in a libgcharm handle; the
opening-angle walk and the force evaluation run on the GPU and lists stay in
HBM unless a caller asks for them (``InteractionLists`` materialises the
reference's per-bucket objects lazily).  Lists built elsewhere (e.g. by the
reference itself) are accepted too and evaluated by the per-work-request kernel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .errors import HeteroRtError
from .generators import ParticleSet, fp32_exact, gen_particles, gen_plummer  # noqa: F401

DEFAULT_SOFTENING = 1e-4


class TreeNode:
    """Read-only view of one node (hr/workloads/nbody.py:52-68)."""

    __slots__ = ("_t", "node_id")

    def __init__(self, tree: "BucketTree", node_id: int):
        self._t = tree
        self.node_id = int(node_id)

    @property
    def center(self):
        return self._t.center[self.node_id]

    @property
    def half_size(self) -> float:
        return float(self._t.half[self.node_id])

    @property
    def size(self) -> float:
        return 2.0 * self.half_size

    @property
    def mass(self) -> float:
        return float(self._t.mass[self.node_id])

    @property
    def com(self):
        return self._t.com[self.node_id]

    @property
    def is_bucket(self) -> bool:
        return bool(self._t.first_child[self.node_id] < 0)

    @property
    def children(self):
        fc = int(self._t.first_child[self.node_id])
        return [] if fc < 0 else [TreeNode(self._t, fc + k) for k in range(int(self._t.n_child[self.node_id]))]

    @property
    def particle_idx(self):
        return self._t.particle_idx(self.node_id)


class BucketTree:
    """Device-resident bucket tree (hr/workloads/nbody.py:71-75)."""

    def __init__(self, ps: ParticleSet, bucket_size: int, forced=None):
        """forced=(levels (m,) int32, prefixes (m, 2) uint64): cubes the build
        splits whatever their count (a rank's part of a distributed tree,
        bh_dist.py)."""
        self.ps = ps
        self.bucket_size = int(bucket_size)
        self.dim = ps.positions.shape[1]
        self.n = ps.positions.shape[0]
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_bh_create", self._ctx.handle, C.byref(self.handle))
        self._gen = 0  # bumps when the handle's list state changes
        self._set(ps, forced, clear_forced=False)

    def _set(self, ps: ParticleSet, forced, clear_forced: bool):
        if forced is not None and len(forced[0]):
            fl = np.ascontiguousarray(forced[0], np.int32)
            fp = np.ascontiguousarray(forced[1], np.uint64).reshape(-1)
            L.call("gc_bh_set_forced_splits", self.handle, len(fl), L.ptr(fl, L.i32p), L.ptr(fp, L.u64p))
        elif clear_forced:
            L.call("gc_bh_set_forced_splits", self.handle, 0, None, None)
        pos, m = L.f64(ps.positions), L.f64(ps.masses)
        L.call("gc_bh_set_particles", self.handle, self.n, self.dim, L.ptr(pos, L.f64p), L.ptr(m, L.f64p),
               float(ps.box), self.bucket_size)
        self._arrays = None

    def reset(self, ps: ParticleSet, forced=None):
        """Rebuild the tree of a new particle set on the same device handle
        (buffers kept: no per-step allocation)."""
        self.ps = ps
        self.dim = ps.positions.shape[1]
        self.n = ps.positions.shape[0]
        self._gen += 1
        self._set(ps, forced, clear_forced=True)

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_bh_destroy(self.handle)
        except Exception:
            pass

    def sizes(self):
        s = np.zeros(5, np.int64)
        L.call("gc_bh_sizes", self.handle, L.ptr(s, L.i64p))
        return s

    def _load(self):
        if self._arrays is None:
            nn, nb = (int(x) for x in self.sizes()[:2])
            d = self.dim
            a = dict(center=np.zeros((nn, d)), half=np.zeros(nn), mass=np.zeros(nn), com=np.zeros((nn, d)),
                     first_child=np.zeros(nn, np.int64), n_child=np.zeros(nn, np.int32),
                     pcount=np.zeros(nn, np.int64), buckets=np.zeros(nb, np.int64), pidx=np.zeros(self.n, np.int64))
            L.call("gc_bh_get_tree", self.handle, L.ptr(a["center"], L.f64p), L.ptr(a["half"], L.f64p),
                   L.ptr(a["mass"], L.f64p), L.ptr(a["com"], L.f64p), L.ptr(a["first_child"], L.i64p),
                   L.ptr(a["n_child"], L.i32p), L.ptr(a["pcount"], L.i64p), L.ptr(a["buckets"], L.i64p),
                   L.ptr(a["pidx"], L.i64p))
            bstart = np.zeros(nn, np.int64)
            bstart[a["buckets"]] = np.concatenate([[0], np.cumsum(a["pcount"][a["buckets"]])[:-1]])
            a["pstart"] = bstart
            self._arrays = a
        return self._arrays

    def __getattr__(self, k):
        if k in ("center", "half", "mass", "com", "first_child", "n_child", "pcount", "pidx", "pstart"):
            return self._load()[k]
        raise AttributeError(k)

    @property
    def bucket_ids(self) -> np.ndarray:
        return self._load()["buckets"]

    @property
    def n_nodes(self) -> int:
        return int(self.sizes()[0])

    def particle_idx(self, node: int) -> np.ndarray:
        a = self._load()
        if a["first_child"][node] >= 0:
            return np.empty(0, np.int64)
        s = a["pstart"][node]
        return a["pidx"][s: s + a["pcount"][node]]

    @property
    def root(self) -> TreeNode:
        return TreeNode(self, 0)

    @property
    def nodes(self):
        return [TreeNode(self, i) for i in range(self.n_nodes)]

    @property
    def buckets(self):
        return [TreeNode(self, int(b)) for b in self.bucket_ids]


def build_bucket_tree(ps: ParticleSet, bucket_size: int) -> BucketTree:
    """hr/workloads/nbody.py:78-120: level-order ids, depth-first buckets,
    float64 mass/COM with the reference's rounding -- built on the GPU
    (csrc/bh_build.cu); there is no host builder in the product."""
    if bucket_size < 1:
        raise ValueError("bucket_size must be >= 1")
    return BucketTree(ps, bucket_size)


@dataclass
class InteractionList:
    bucket_id: int
    node_interactions: list
    particle_interactions: list
    walk_order: list
    item_count: int


class InteractionLists:
    """Device lists of one walk (CSR over buckets in DFS order); behaves as the
    reference's ``list[InteractionList]`` (materialised on first access)."""

    def __init__(self, tree: BucketTree, theta: float):
        self.tree = tree
        self.theta = float(theta)
        self._gen = tree._gen
        self._csr = None
        self._objs = None

    def csr(self):
        """(ptr, ids, kind, item_count): kind 0 = node, 1 = particle entry."""
        if self._csr is None:
            t = self.tree
            _ensure_walk(t, self)
            nb = len(t.bucket_ids)
            ent = int(t.sizes()[2])
            ptr = np.zeros(nb + 1, np.int64)
            ids = np.zeros(ent, np.int64)
            kind = np.zeros(ent, np.int8)
            ic = np.zeros(nb, np.int64)
            L.call("gc_bh_get_lists", t.handle, L.ptr(ptr, L.i64p), L.ptr(ids, L.i64p), L.ptr(kind, L.i8p),
                   L.ptr(ic, L.i64p))
            self._csr = (ptr, ids, kind, ic)
        return self._csr

    @property
    def item_count(self) -> np.ndarray:
        return self.csr()[3]

    def _materialise(self):
        if self._objs is None:
            ptr, ids, kind, ic = self.csr()
            objs = []
            for b, bid in enumerate(self.tree.bucket_ids):
                s = slice(ptr[b], ptr[b + 1])
                w, k = ids[s], kind[s]
                objs.append(InteractionList(int(bid), w[k == 0].tolist(), w[k == 1].tolist(), w.tolist(),
                                            int(ic[b])))
            self._objs = objs
        return self._objs

    def __len__(self):
        return len(self.tree.bucket_ids)

    def __getitem__(self, i):
        return self._materialise()[i]

    def __iter__(self):
        return iter(self._materialise())


def _ensure_walk(tree: BucketTree, lists: InteractionLists):
    if lists._gen != tree._gen:
        L.call("gc_bh_walk", tree.handle, lists.theta)
        tree._gen += 1
        lists._gen = tree._gen


def build_interaction_lists(tree: BucketTree, theta: float, ps: ParticleSet | None = None) -> InteractionLists:
    """hr/workloads/nbody.py:160-199 on the GPU (float64 decisions, bit-exact)."""
    if theta < 0:
        raise ValueError("theta must be >= 0")
    L.call("gc_bh_walk", tree.handle, float(theta))
    tree._gen += 1
    lists = InteractionLists(tree, theta)
    lists._gen = tree._gen
    return lists


def lists_to_csr(lists):
    """Reference-style list[InteractionList] -> (ptr, ids, kind)."""
    ptr = np.zeros(len(lists) + 1, np.int64)
    ids, kind = [], []
    for i, il in enumerate(lists):
        nodes = set(il.node_interactions)
        ids.extend(il.walk_order)
        kind.extend(0 if b in nodes else 1 for b in il.walk_order)
        ptr[i + 1] = len(ids)
    return ptr, np.asarray(ids, np.int64), np.asarray(kind, np.int8)


def eval_forces(tree: BucketTree, lists, ps: ParticleSet | None = None, g: float = 1.0,
                eps: float = DEFAULT_SOFTENING) -> np.ndarray:
    """hr/workloads/nbody.py:216-250: forces implied by the interaction lists
    (float64 (n, dim), original particle order)."""
    if ps is not None and ps is not tree.ps and not (
            np.array_equal(ps.positions, tree.ps.positions) and np.array_equal(ps.masses, tree.ps.masses)):
        raise ValueError("eval_forces: particle set differs from the one the tree was built on")
    if isinstance(lists, InteractionLists) and lists.tree is tree:
        _ensure_walk(tree, lists)
    else:
        if isinstance(lists, tuple):
            ptr, ids, kind = lists[:3]
        else:
            ptr, ids, kind = lists_to_csr(lists)
        ptr, ids, kind = L.i64(ptr), L.i64(ids), np.ascontiguousarray(kind, np.int8)
        L.call("gc_bh_set_lists", tree.handle, len(ptr) - 1, L.ptr(ptr, L.i64p), L.ptr(ids, L.i64p),
               L.ptr(kind, L.i8p))
        tree._gen += 1
    out = np.zeros((tree.n, tree.dim))
    L.call("gc_bh_forces", tree.handle, float(g), float(eps), L.ptr(out, L.f64p))
    return out


def eval_forces_potential(tree: BucketTree, lists: "InteractionLists", g: float = 1.0,
                          eps: float = DEFAULT_SOFTENING):
    """Forces (as eval_forces) plus per-particle potential energy
    -g m_i sum_j m_j / sqrt(r^2 + eps^2) over the same lists (no reference
    counterpart; the oracle restates it beside forces_from_points,
    hr/kernels.py:70-88).  Device lists only."""
    if not (isinstance(lists, InteractionLists) and lists.tree is tree):
        raise ValueError("eval_forces_potential: needs the tree's own device lists")
    _ensure_walk(tree, lists)
    f, pot = np.zeros((tree.n, tree.dim)), np.zeros(tree.n)
    L.call("gc_bh_forces_potential", tree.handle, float(g), float(eps), L.ptr(f, L.f64p), L.ptr(pot, L.f64p))
    return f, pot


def interactions(tree: BucketTree) -> int:
    """Sum over buckets of n_b * item_count_b for the current lists."""
    out = np.zeros(1, np.int64)
    L.call("gc_bh_interactions", tree.handle, L.ptr(out, L.i64p))
    return int(out[0])


def periodic_forces(tree: BucketTree, theta: float, nrep: int = 1, g: float = 1.0,
                    eps: float = DEFAULT_SOFTENING):
    """Periodic Barnes-Hut forces: every bucket walks the
    tree once per image of the box ((2 nrep + 1)^3 images, the box of the
    tree; nrep <= 1), the sources of image s at their position + s.  The long-range
    remainder beyond the images is the ewald kernel class (ewald.py).
    Returns (forces (n, 3), per-bucket entries, per-bucket items)."""
    L.call("gc_bh_set_periodic", tree.handle, int(nrep), float(tree.ps.box))
    try:
        L.call("gc_bh_walk", tree.handle, float(theta))
        out = np.zeros((tree.n, tree.dim))
        L.call("gc_bh_forces", tree.handle, float(g), float(eps), L.ptr(out, L.f64p))
        nb = int(tree.sizes()[1])
        ptr, ic = np.zeros(nb + 1, np.int64), np.zeros(nb, np.int64)
        L.call("gc_bh_get_lists", tree.handle, L.ptr(ptr, L.i64p), None, None, L.ptr(ic, L.i64p))
    finally:
        L.call("gc_bh_set_periodic", tree.handle, 0, 0.0)
        tree._gen += 1
    return out, np.diff(ptr), ic


def direct_force_oracle(ps: ParticleSet, g: float = 1.0, eps: float = DEFAULT_SOFTENING) -> np.ndarray:
    """hr/workloads/nbody.py:202-213 on the GPU (exact float64 pair sums)."""
    from . import kernels
    if eps == 0.0:
        _, counts = np.unique(ps.positions, axis=0, return_counts=True)
        if (counts > 1).any():
            raise HeteroRtError("coincident particles with zero softening")
    return kernels.direct_forces(ps.positions, ps.masses, g, eps)


class BHStep:
    """End-to-end step through the C ABI (host buffers in, host forces out):
    H2D particles, tree, device walk, forces, D2H (gc_bh_step)."""

    def __init__(self, bucket_size=8, theta=0.7, g=1.0, eps=DEFAULT_SOFTENING):
        self.bucket_size, self.theta, self.g, self.eps = bucket_size, theta, g, eps
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_bh_create", self._ctx.handle, C.byref(self.handle))

    def __call__(self, positions, masses, box=1.0, out=None):
        pos, m = L.f64(positions), L.f64(masses)
        n, d = pos.shape
        if out is None:
            out = np.zeros((n, d))
        L.call("gc_bh_step", self.handle, n, d, L.ptr(pos, L.f64p), L.ptr(m, L.f64p), float(box),
               int(self.bucket_size), float(self.theta), float(self.g), float(self.eps), L.ptr(out, L.f64p))
        return out

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_bh_destroy(self.handle)
        except Exception:
            pass
