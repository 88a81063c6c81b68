"""Distributed Barnes-Hut over the GPUs of one box: partitioned trees and a
locally-essential-tree (LET) exchange (SURVEY.md §8e, configs[3]).

The reference runs one process (hr/workloads/nbody.py:78-250).  Here every
rank owns a contiguous range of the GLOBAL depth-first (octant-key) order and
never holds the whole particle set, yet each rank's interaction lists are
bit-identical to the ones a single GPU builds over all particles:

1. keys + sample sort.  Octant keys of the reference's descent
   (nbody.py:97-108, ``gc_bh_keys``); splitters from an all-gathered sample;
   particles move with one all-to-all (NCCL on GPUs, gloo in the CPU tests).
2. straddling cubes.  The cubes that contain particles of two ranks are the
   common-prefix cubes of each boundary pair.  Their global populations
   (all-reduce) must exceed the bucket size (the global tree splits them); a
   boundary that would cut a global bucket is moved past it and step 1 redone.
3. local subtrees.  Each rank builds its particles' tree on the device with
   the straddling cubes forced to split (``gc_bh_set_forced_splits``): every
   other node is complete and identical to the global tree's (same particles,
   same float64 sums).  Its maximal complete nodes are the rank's BRANCH
   nodes.
4. top of the tree.  Branch summaries are all-gathered; every rank computes
   the straddling nodes' mass / centre of mass in the reference's child order
   (``_fill_mass``, nbody.py:123-135).
5. LET.  For every peer, each rank walks its subtrees against the peer's
   bucket bounding box: a node the box accepts (``size / d < theta`` with d
   the distance to the box, a lower bound of the distance to every bucket
   inside it, nbody.py:155-178, with a 1e-9 margin) is all the peer needs;
   otherwise its children (or an opened bucket's particles) are sent.  The
   fetch list is exactly the data manager's ``missing`` set of remote nodes
   (hr/memory.py:328-338) for the peer's whole bucket range, computed
   sender-side so one all-to-all moves it.
6. assembly + step.  Top nodes, all branches, the own subtrees and the
   received LET nodes form one tree in global level order
   (``gc_bh_set_tree``); a remote node no own bucket may open is sealed (a
   poisoned bucket: opening it would give NaN forces).  The own buckets form
   whole walk groups; walk + forces run on them only.

The device kernels and the C-ABI are those of the one-GPU path; the host code
here is index bookkeeping over summaries (no force or list arithmetic).
Collectives go through ``Comm`` (torch.distributed; the CPU tests use gloo and
run the same protocol with the float64 oracle as the per-rank backend).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

NLEV_MAX = 42
_M63 = (1 << 63) - 1


# --------------------------------------------------------------------------
# keys: 126-bit ints K = k1 << 63 | k2, level l digit at bit D(l)
# --------------------------------------------------------------------------
def _dpos(level: int) -> int:
    return 63 + 3 * (20 - level) if level < 21 else 3 * (41 - level)


def _mask(level: int) -> int:
    """Bits of the digits of levels < level."""
    m = 0
    for l in range(level):
        m |= 7 << _dpos(l)
    return m


_MASKS = [_mask(L) for L in range(NLEV_MAX + 1)]
_FULL = _MASKS[NLEV_MAX]


def _split(K: int):
    return np.uint64(K >> 63), np.uint64(K & _M63)


def _join(a, b) -> int:
    return (int(a) << 63) | int(b)


def common_levels(Ka: int, Kb: int, nlev: int) -> int:
    """Number of leading digits two keys share (the deepest common cube's level)."""
    L = 0
    while L < nlev and ((Ka >> _dpos(L)) & 7) == ((Kb >> _dpos(L)) & 7):
        L += 1
    return L


def n_levels(box: float) -> int:
    """Levels at which a node may still split (half >= 1e-9, nbody.py:94)."""
    n, h = 0, box / 2.0
    while h >= 1e-9 and n <= NLEV_MAX:
        n += 1
        h /= 2.0
    return n


def lex_search(k1, k2, a1, a2, side="left") -> int:
    """Position of (a1, a2) in arrays sorted by (k1, k2)."""
    i0 = int(np.searchsorted(k1, a1, "left"))
    i1 = int(np.searchsorted(k1, a1, "right"))
    return i0 + int(np.searchsorted(k2[i0:i1], a2, side))


def cube_range(k1, k2, level: int, P: int):
    """[lo, hi) of the sorted keys inside cube (level, P)."""
    lo = lex_search(k1, k2, *_split(P), "left")
    hi = lex_search(k1, k2, *_split(P | (_FULL & ~_MASKS[level])), "right")
    return lo, hi


# --------------------------------------------------------------------------
# host-orchestration helpers: the protocol's million-row sorts and gathers run
# on the GPU when one is present (numpy costs ~0.5 s per 1M-row lexsort);
# small arrays and CPU-only runs keep numpy
# --------------------------------------------------------------------------
_DEV_ROWS = 1 << 16


def _on_gpu(n: int) -> bool:
    if n < _DEV_ROWS:
        return False
    try:
        import torch
        return torch.cuda.is_available()
    except ImportError:  # pragma: no cover
        return False


def _gpu():
    """The library context's device (the rank's GPU), as a torch device."""
    import torch
    from . import _lib as L
    return torch.device("cuda", L.context().device % torch.cuda.device_count())


def _as_i64(k: np.ndarray):
    """A sort key as int64 with the same order, or None (uint64 with the top bit set)."""
    k = np.ascontiguousarray(k)
    if k.dtype == np.uint64:
        return None if np.any(k >> np.uint64(63)) else k.view(np.int64)
    if k.dtype == np.bool_:
        return k.astype(np.int64)
    return k.astype(np.int64, copy=False)


def _lexsort(keys) -> np.ndarray:
    """np.lexsort(keys) (the last key is the primary one): stable LSD passes of
    torch.argsort on the GPU for large inputs."""
    n = len(keys[0])
    if not _on_gpu(n):
        return np.lexsort(keys)
    ks = [_as_i64(k) for k in keys]
    if any(k is None for k in ks):
        return np.lexsort(keys)
    import torch
    dev = _gpu()
    o = None
    for k in ks:
        t = torch.from_numpy(k).to(dev)
        o = torch.argsort(t, stable=True) if o is None else o[torch.argsort(t[o], stable=True)]
    return o.cpu().numpy()


def _take(o: np.ndarray, *arrays):
    """Row gathers a[o] for each array (GPU for large inputs)."""
    if not _on_gpu(len(o)):
        return tuple(a[o] for a in arrays)
    import torch
    dev = _gpu()
    ot = torch.from_numpy(np.ascontiguousarray(o, np.int64)).to(dev)
    out = []
    for a in arrays:
        a = np.ascontiguousarray(a)
        raw = a.dtype == np.uint64
        t = torch.from_numpy(a.view(np.int64) if raw else a).to(dev)
        r = t[ot].cpu().numpy()
        out.append(r.view(np.uint64) if raw else r)
    return tuple(out)


def _key16(lvl, p1, p2) -> np.ndarray:
    """Sortable bytes of (level, prefix) for vectorised searches (big endian)."""
    a = np.empty(len(lvl), dtype=[("l", ">u2"), ("a", ">u8"), ("b", ">u8")])
    a["l"], a["a"], a["b"] = lvl, p1, p2
    return a.view("S18").ravel()


# --------------------------------------------------------------------------
# collectives
# --------------------------------------------------------------------------
class Comm:
    """The collectives of the protocol over a torch.distributed group (NCCL:
    device tensors; gloo: host tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def _t(self, a: np.ndarray):
        import torch
        return torch.as_tensor(np.ascontiguousarray(a)).to(self.device)

    def allgather(self, a: np.ndarray) -> list:
        """Variable-length all-gather of a 1-D (or row-major 2-D) array."""
        import torch
        a = np.ascontiguousarray(a)
        row = a.shape[1:]
        n = self._t(np.array([a.shape[0]], np.int64))
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        m = max(ns + [1])
        buf = np.zeros((m,) + row, a.dtype)
        buf[: a.shape[0]] = a
        t = self._t(buf.view(np.uint8) if a.dtype == np.uint64 else buf)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        res = []
        for k, o in enumerate(outs):
            v = o.cpu().numpy()
            if a.dtype == np.uint64:
                v = v.view(np.uint64).reshape((m,) + row)
            res.append(v[: ns[k]])
        return res

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(np.ascontiguousarray(a, np.int64))
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def alltoallv(self, parts: list) -> list:
        """parts[r] (rows of equal shape / dtype) goes to rank r; returns what
        every rank sent here."""
        import torch
        dt = parts[0].dtype
        row = parts[0].shape[1:]
        raw = dt == np.uint64
        send_n = np.array([p.shape[0] for p in parts], np.int64)
        sn = self._t(send_n)
        rn = torch.empty_like(sn)
        self.dist.all_to_all_single(rn, sn, group=self.group)
        recv_n = rn.cpu().numpy()
        per = int(np.prod(row)) if row else 1
        flat = np.concatenate([np.ascontiguousarray(p).reshape(-1) for p in parts]) if parts else np.zeros(0, dt)
        if raw:
            flat = flat.view(np.int64)
        st = self._t(flat)
        rt = torch.empty(int(recv_n.sum()) * per, dtype=st.dtype, device=st.device)
        self.dist.all_to_all_single(rt, st, [int(x) * per for x in recv_n], [int(x) * per for x in send_n],
                                    group=self.group)
        out = rt.cpu().numpy()
        if raw:
            out = out.view(np.uint64)
        res, o = [], 0
        for k in range(self.world):
            c = int(recv_n[k]) * per
            res.append(out[o: o + c].reshape((int(recv_n[k]),) + row))
            o += c
        return res


# --------------------------------------------------------------------------
# backends: the per-rank device work (product) -- the CPU tests substitute
# the float64 oracle (oracle/dist_backend.py)
# --------------------------------------------------------------------------
class DeviceBackend:
    """libgcharm.so: keys, the forced-split local build, the assembled-tree step.
    ``last`` holds the device times (CUDA events, ms) of the last step's walk
    and force kernels and its interaction count."""

    def __init__(self):
        self.last = {}
        self._local = None  # BucketTree reused across steps (its device buffers stay allocated)
        self._h = None  # handle of the assembled tree, reused across steps

    def __del__(self):
        try:
            if self._h is not None:
                from . import _lib as L
                L.load().gc_bh_destroy(self._h)
        except Exception:
            pass

    def keys(self, pos, box):
        from . import _lib as L
        ctx = L.context()
        pos = L.f64(pos)
        n, dim = pos.shape
        k1, k2 = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        L.call("gc_bh_keys", ctx.handle, n, dim, L.ptr(pos, L.f64p), float(box), L.ptr(k1, L.u64p),
               L.ptr(k2, L.u64p))
        return k1, k2

    def local_tree(self, pos, mass, bucket, box, forced):
        from . import nbody
        from .generators import ParticleSet
        ps = ParticleSet(pos, mass, np.zeros_like(pos), box)
        t = self._local
        if t is None or t.bucket_size != int(bucket):
            t = self._local = nbody.BucketTree(ps, bucket, forced=forced)
        else:
            t.reset(ps, forced)
        a = dict(t._load())
        a["buckets"] = np.asarray(t.bucket_ids)
        return a

    def step(self, tree: dict, own: tuple, theta: float, g: float, eps: float, want_lists: bool):
        """Walk + forces of the own buckets [own[0], own[1]) of an assembled
        tree; returns (forces of every particle row, lists CSR or None)."""
        from . import _lib as L
        ctx = L.context()
        if self._h is None:
            self._h = C.c_void_p()
            L.call("gc_bh_create", ctx.handle, C.byref(self._h))
        h = self._h
        # the handle is kept across steps: gc_bh_set_tree resets every per-tree state
        n = len(tree["pmass"])
        nn = len(tree["half"])
        dim = tree["center"].shape[1]
        cuts = np.array(own, np.int64)
        ar = {k: np.ascontiguousarray(v) for k, v in tree.items()}
        L.call("gc_bh_set_tree", h, nn, dim, float(tree["box"]), int(tree["bucket"]),
               L.ptr(L.f64(ar["center"]), L.f64p), L.ptr(L.f64(ar["half"]), L.f64p),
               L.ptr(L.f64(ar["mass"]), L.f64p), L.ptr(L.f64(ar["com"]), L.f64p),
               L.ptr(L.i64(ar["first_child"]), L.i64p), L.ptr(np.ascontiguousarray(ar["n_child"], np.int32),
                                                               L.i32p),
               L.ptr(L.i64(ar["pstart"]), L.i64p), L.ptr(L.i64(ar["pcount"]), L.i64p),
               len(ar["buckets"]), L.ptr(L.i64(ar["buckets"]), L.i64p), n, L.ptr(L.i64(ar["order"]), L.i64p),
               L.ptr(L.f64(ar["pos"]), L.f64p), L.ptr(L.f64(ar["pmass"]), L.f64p), len(cuts),
               L.ptr(cuts, L.i64p))
        ng = np.zeros(1, np.int64)
        L.call("gc_bh_groups", h, L.ptr(ng, L.i64p), None)
        wfb = np.zeros(int(ng[0]) + 1, np.int64)
        L.call("gc_bh_groups", h, L.ptr(ng, L.i64p), L.ptr(wfb, L.i64p))
        g0, g1 = int(np.searchsorted(wfb, own[0])), int(np.searchsorted(wfb, own[1]))
        assert wfb[g0] == own[0] and wfb[g1] == own[1], "own buckets must form whole walk groups"
        L.call("gc_bh_set_range", h, g0, g1)
        L.call("gc_bh_walk", h, float(theta))  # stats walk (sizes the union pool for this tree)
        L.call("gc_bh_walk", h, float(theta))
        L.call("gc_bh_forces_async", h, float(g), float(eps))
        tm = np.zeros(3)
        L.call("gc_bh_timings", h, L.ptr(tm, L.f64p))
        f = np.zeros((n, dim))
        L.call("gc_bh_get_forces", h, L.ptr(f, L.f64p))
        cnt = np.zeros(1, np.int64)
        L.call("gc_bh_interactions", h, L.ptr(cnt, L.i64p))
        self.last = dict(walk_ms=float(tm[0]), force_ms=float(tm[1]), interactions=int(cnt[0]))
        lists = None
        if want_lists:
            nb = len(ar["buckets"])
            ptr, ic = np.zeros(nb + 1, np.int64), np.zeros(nb, np.int64)
            L.call("gc_bh_get_lists", h, L.ptr(ptr, L.i64p), None, None, L.ptr(ic, L.i64p))
            ids, kind = np.zeros(int(ptr[-1]), np.int64), np.zeros(int(ptr[-1]), np.int8)
            L.call("gc_bh_get_lists", h, L.ptr(ptr, L.i64p), L.ptr(ids, L.i64p), L.ptr(kind, L.i8p),
                   L.ptr(ic, L.i64p))
            lists = (ptr, ids, kind, ic)
        return f, lists


# --------------------------------------------------------------------------
# the protocol
# --------------------------------------------------------------------------
@dataclass
class DistResult:
    gid: np.ndarray  # global ids of this rank's particles (its DFS range)
    forces: np.ndarray  # (n_local, dim), rows of gid
    tree: dict  # the assembled tree (level, prefix per node for list mapping)
    own: tuple  # own bucket range (DFS indices of the assembled tree)
    lists: tuple | None = None  # CSR over the assembled tree's buckets (own range filled)
    stats: dict = field(default_factory=dict)


def _node_prefixes(t: dict):
    """Level and key prefix of every node of a tree in the reference layout."""
    nn = len(t["half"])
    center = t["center"]
    dim = center.shape[1]
    lvl = np.zeros(nn, np.int64)
    p1 = np.zeros(nn, np.uint64)
    p2 = np.zeros(nn, np.uint64)
    fc, nc = t["first_child"], t["n_child"]
    front = np.array([0], np.int64)
    L = 0
    while len(front):
        par = front[fc[front] >= 0]
        if not len(par):
            break
        cnt = nc[par].astype(np.int64)
        kids = np.repeat(fc[par], cnt) + (np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt))
        pp = np.repeat(par, cnt)
        q = np.zeros(len(kids), np.uint64)
        for k in range(dim):
            q |= (center[kids, k] > center[pp, k]).astype(np.uint64) << np.uint64(k)
        lvl[kids] = L + 1
        if L < 21:
            p1[kids] = p1[pp] | (q << np.uint64(3 * (20 - L)))
            p2[kids] = p2[pp]
        else:
            p1[kids] = p1[pp]
            p2[kids] = p2[pp] | (q << np.uint64(3 * (41 - L)))
        front = kids
        L += 1
    return lvl, p1, p2


def _cube_center(level: int, P: int, box: float, dim: int):
    """Centre of cube (level, P) by the reference's halving sequence (nbody.py:105-108)."""
    c = [box / 2.0] * dim
    h = box / 2.0
    for l in range(level):
        q = (P >> _dpos(l)) & 7
        ch = h / 2.0
        for k in range(dim):
            c[k] = c[k] + (ch if (q >> k) & 1 else -ch)
        h = ch
    return c, h


class DistBH:
    """One Barnes-Hut step over a particle set partitioned across the ranks of
    ``comm`` (configs[3]); the reference API's parameters (bucket_size,
    theta, g, eps: hr/workloads/nbody.py:23, 216)."""

    def __init__(self, comm, bucket_size=8, theta=0.7, g=1.0, eps=1e-4, box=1.0, backend=None, sample=256,
                 shares=None, balance=True):
        """shares: fixed particle shares per rank (default: equal, then --
        with balance -- the measured speeds of the previous steps).  The
        reference's adaptive CPU/GPU split (hr/scheduler.py, scheduler.KWayEstimate)
        over the ranks: each step's device walk + force time per own particle
        is all-gathered, and the next partition cuts the key order at the
        speed-proportional cumulative shares.  Lists and forces do not depend
        on where the boundaries fall."""
        from . import scheduler as sch
        self.comm = comm
        self.bucket = int(bucket_size)
        self.theta, self.g, self.eps, self.box = float(theta), float(g), float(eps), float(box)
        self.backend = backend or DeviceBackend()
        self.sample = sample
        self.stats = {}
        self.fixed_shares = None if shares is None else [float(x) for x in shares]
        if self.fixed_shares is not None and (len(self.fixed_shares) != comm.world or
                                              abs(sum(self.fixed_shares) - 1.0) > 1e-9 or
                                              min(self.fixed_shares) <= 0.0):
            raise ValueError("shares: one positive share per rank, summing to 1")
        self.balance = sch.KWayEstimate(comm.world) if balance else None

    def shares(self):
        """Particle shares of the next partition."""
        if self.fixed_shares is not None:
            return list(self.fixed_shares)
        if self.balance is not None:
            return self.balance.shares()
        return [1.0 / self.comm.world] * self.comm.world

    # ---- 1 + 2: keys, sample sort, straddling cubes ----------------------------
    def _partition(self, pos, mass, gid):
        cm, box = self.comm, self.box
        nlev = n_levels(box)
        k1, k2 = self.backend.keys(pos, box)
        o = _lexsort((gid, k2, k1))
        pos, mass, gid, k1, k2 = _take(o, pos, mass, gid, k1, k2)
        # splitters: world - 1 quantiles of an all-gathered sample of (key, gid)
        n = len(gid)
        take = np.unique(np.linspace(0, max(n - 1, 0), min(n, self.sample)).astype(np.int64)) if n else np.zeros(0, int)
        smp = np.stack([k1[take].view(np.int64), k2[take].view(np.int64), gid[take]], axis=1) if n else np.zeros((0, 3), np.int64)
        allsmp = np.concatenate(cm.allgather(smp))
        allsmp = allsmp[np.lexsort((allsmp[:, 2], allsmp[:, 1].view(np.uint64), allsmp[:, 0].view(np.uint64)))]
        splitters = []
        shares = self.shares()
        equal = all(abs(x - 1.0 / cm.world) < 1e-12 for x in shares)
        cum = np.cumsum(shares)
        for r in range(1, cm.world):
            # the sample quantile at the cumulative share of ranks < r
            j = (r * len(allsmp)) // cm.world if equal else int(cum[r - 1] * len(allsmp))
            s = allsmp[min(j, len(allsmp) - 1)]
            splitters.append((_join(np.uint64(s[0]), np.uint64(s[1])), int(s[2])))
        for it in range(64):
            dest = np.zeros(len(gid), np.int64)
            for (K, sg) in splitters:
                s1, s2 = _split(K)
                dest += (k1 > s1) | ((k1 == s1) & ((k2 > s2) | ((k2 == s2) & (gid >= sg))))
            cut = np.searchsorted(dest, np.arange(cm.world + 1), "left")  # rows are sorted: dest is monotone
            recv_pos = cm.alltoallv([pos[cut[r]:cut[r + 1]] for r in range(cm.world)])
            recv_m = cm.alltoallv([mass[cut[r]:cut[r + 1]] for r in range(cm.world)])
            recv_g = cm.alltoallv([gid[cut[r]:cut[r + 1]] for r in range(cm.world)])
            recv_k1 = cm.alltoallv([k1[cut[r]:cut[r + 1]] for r in range(cm.world)])
            recv_k2 = cm.alltoallv([k2[cut[r]:cut[r + 1]] for r in range(cm.world)])
            pos, mass, gid = np.concatenate(recv_pos), np.concatenate(recv_m), np.concatenate(recv_g)
            k1, k2 = np.concatenate(recv_k1), np.concatenate(recv_k2)
            o = _lexsort((gid, k2, k1))
            pos, mass, gid, k1, k2 = _take(o, pos, mass, gid, k1, k2)
            # boundaries between consecutive non-empty ranks
            ends = np.array([[len(gid), _join(k1[0], k2[0]) >> 63 if len(gid) else 0,
                              _join(k1[0], k2[0]) & _M63 if len(gid) else 0,
                              _join(k1[-1], k2[-1]) >> 63 if len(gid) else 0,
                              _join(k1[-1], k2[-1]) & _M63 if len(gid) else 0]], np.uint64)
            ends = np.concatenate(cm.allgather(ends))
            cubes = {}  # (level, P) -> (rank before, rank after) of its boundary (for the fix-up)
            prev = None
            for r in range(cm.world):
                if int(ends[r, 0]) == 0:
                    continue
                if prev is not None:
                    Ka = _join(ends[prev, 3], ends[prev, 4])
                    Kb = _join(ends[r, 1], ends[r, 2])
                    Lc = common_levels(Ka, Kb, NLEV_MAX)
                    for L in range(Lc + 1):
                        cubes.setdefault((L, Ka & _MASKS[L]), (prev, r))
                prev = r
            keys_ = sorted(cubes)
            local = np.array([cube_range(k1, k2, L, P) for (L, P) in keys_], np.int64).reshape(-1, 2)
            cnt = cm.allreduce_sum(local[:, 1] - local[:, 0]) if len(keys_) else np.zeros(0, np.int64)
            bad = [(L, P) for (L, P), c in zip(keys_, cnt) if c <= self.bucket or L >= nlev]
            if not bad:
                break
            # a global bucket (or an unsplittable cube) would straddle: move the
            # boundary past the shallowest offending cube, redo the exchange
            L, P = min(bad)
            a, b = cubes[(L, P)]
            end = ((P | (_FULL & ~_MASKS[L])) + 1, -1)  # first key after the cube
            splitters = [max(sp, end) if i >= a else sp for i, sp in enumerate(splitters)]
        else:
            raise RuntimeError("boundary fix-up did not converge")
        self.stats["partition_iterations"] = it + 1
        return pos, mass, gid, k1, k2, keys_, cnt

    # ---- the step ---------------------------------------------------------------
    def step(self, pos, mass, gid, want_lists=False) -> DistResult:
        """Forces on this rank's particles (of the global N-body system whose
        other particles the other ranks hold); pos/mass/gid: any initial share."""
        import time
        tic = [time.perf_counter()]

        def lap(name):
            tic.append(time.perf_counter())
            self.stats["t_" + name] = tic[-1] - tic[-2]

        cm, box = self.comm, self.box
        pos = np.ascontiguousarray(pos, np.float64)
        dim = pos.shape[1]
        mass = np.ascontiguousarray(mass, np.float64)
        gid = np.ascontiguousarray(gid, np.int64)
        pos, mass, gid, k1, k2, scubes, scount = self._partition(pos, mass, gid)
        lap("partition")
        n = len(gid)
        if not n:
            raise ValueError("a rank holds no particles after the partition (fewer particles than ranks?)")
        # local ids in ascending global id: buckets keep ascending particle_idx
        # (nbody.py:110), so sums over a bucket's particles run in the
        # single-process order
        o = _lexsort((gid,))
        pos, mass, gid = _take(o, pos, mass, gid)
        forced = (np.array([L for L, _ in scubes], np.int32),
                  np.array([[P >> 63, P & _M63] for _, P in scubes], np.uint64).reshape(-1, 2))
        # ---- 3: own subtrees ------------------------------------------------
        if n:
            t = self.backend.local_tree(pos, mass, self.bucket, box, forced)
            lvl, p1, p2 = _node_prefixes(t)
            nn = len(lvl)
            if scubes:
                sk = np.sort(_key16(forced[0], forced[1][:, 0], forced[1][:, 1]))
                nk = _key16(lvl, p1, p2)
                j = np.minimum(np.searchsorted(sk, nk), len(sk) - 1)
                is_strad = sk[j] == nk
            else:
                is_strad = np.zeros(nn, bool)
            parent = np.full(nn, -1, np.int64)
            hasc = t["first_child"] >= 0
            cnt_c = t["n_child"][hasc].astype(np.int64)
            kid = np.repeat(t["first_child"][hasc], cnt_c) + (
                np.arange(cnt_c.sum()) - np.repeat(np.cumsum(cnt_c) - cnt_c, cnt_c))
            parent[kid] = np.repeat(np.nonzero(hasc)[0], cnt_c)
            branch = ~is_strad & ((parent < 0) | is_strad[np.maximum(parent, 0)])
            branch[0] = not is_strad[0]
            own_node = ~is_strad  # complete local nodes (global tree nodes)
        else:
            t, nn = None, 0
        lap("local_tree")
        # ---- 4: branch summaries, top of the tree ------------------------------
        bcols = 7 + 2 * dim  # level, p1, p2, half, mass, is_bucket, count, center(dim), com(dim)
        if n:
            bi = np.nonzero(branch)[0]
            br = np.zeros((len(bi), bcols))
            br[:, 0] = lvl[bi]
            br[:, 1] = p1[bi].view(np.float64)
            br[:, 2] = p2[bi].view(np.float64)
            br[:, 3] = t["half"][bi]
            br[:, 4] = t["mass"][bi]
            br[:, 5] = (t["first_child"][bi] < 0)
            br[:, 6] = t["pcount"][bi]
            br[:, 7:7 + dim] = t["center"][bi]
            br[:, 7 + dim:] = t["com"][bi]
        else:
            br = np.zeros((0, bcols))
        allbr = cm.allgather(br)
        aabb = np.full((1, 2 * dim), np.nan)
        if n:
            bk = t["buckets"]
            lo_ = t["center"][bk] - t["half"][bk][:, None]
            hi_ = t["center"][bk] + t["half"][bk][:, None]
            aabb[0, :dim] = lo_.min(axis=0)
            aabb[0, dim:] = hi_.max(axis=0)
        aabbs = [a[0] for a in cm.allgather(aabb)]
        top = self._top_nodes(scubes, allbr, dim)
        lap("top")
        # ---- 5: LET for every peer ------------------------------------------
        let_nodes, let_parts = [], []
        for r in range(cm.world):
            if r == cm.rank or not n or np.isnan(aabbs[r][0]):
                let_nodes.append(np.zeros((0, 8 + 2 * dim)))
                let_parts.append(np.zeros((0, dim + 2)))
                continue
            a, b = self._let_for(t, lvl, p1, p2, branch, pos, mass, gid, aabbs[r], dim)
            let_nodes.append(a)
            let_parts.append(b)
        rn = cm.alltoallv(let_nodes)
        rp = cm.alltoallv(let_parts)
        lap("let")
        # ---- 6: assemble, walk the own buckets ----------------------------------
        tree, own, stats = self._assemble(t, lvl, p1, p2, own_node if n else None, pos, mass, gid, top, allbr, rn,
                                          rp, dim)
        self.stats.update(stats)
        lap("assemble")
        f, lists = self.backend.step(tree, own, self.theta, self.g, self.eps, want_lists)
        lap("device_step")
        self._record_speed(n)
        return DistResult(gid=gid, forces=f[:n], tree=tree, own=own, lists=lists, stats=dict(self.stats))

    def _record_speed(self, n_own: int):
        """All-gather this step's device walk + force time per own particle
        into the balancer (every rank records the same samples)."""
        last = getattr(self.backend, "last", None) or {}
        if self.balance is None or "walk_ms" not in last:
            return
        ms = float(last["walk_ms"]) + float(last["force_ms"])
        rows = self.comm.allgather(np.array([[ms, float(n_own)]]))
        for r, row in enumerate(rows):
            if len(row) and row[0, 0] > 0.0 and row[0, 1] >= 1.0:
                self.balance.record(r, int(row[0, 1]), float(row[0, 0]))
        self.stats["shares_next"] = [round(x, 4) for x in self.balance.shares()]

    def _top_nodes(self, scubes, allbr, dim):
        """Straddling nodes with the reference's mass / COM sums over children in octant order."""
        box = self.box
        rows = {}
        for br in allbr:
            for row in br:
                L = int(row[0])
                P = _join(np.float64(row[1]).view(np.uint64), np.float64(row[2]).view(np.uint64))
                rows[(L, P)] = (row[4], row[7 + dim: 7 + 2 * dim])
        top = {}
        for (L, P) in sorted(scubes, key=lambda x: -x[0]):
            kids = []
            for q in range(1 << dim):
                Q = P | (q << _dpos(L))
                if (L + 1, Q) in top:
                    kids.append(top[(L + 1, Q)][:2])
                elif (L + 1, Q) in rows:
                    kids.append(rows[(L + 1, Q)])
            m = 0.0
            com = np.zeros(dim)
            for cm_, cc in kids:
                m += cm_
                for k in range(dim):
                    com[k] = com[k] + cc[k] * cm_
            com = com / m
            c, h = _cube_center(L, P, box, dim)
            top[(L, P)] = (m, com, np.array(c), h)
        return top

    def _let_for(self, t, lvl, p1, p2, branch, pos, mass, gid, box_p, dim):
        """Nodes (and opened buckets' particles) of this rank's subtrees that the
        peer with bucket box `box_p` needs: rows (level, p1, p2, kind, half, mass,
        pcount, _, center, com) with kind 0 = accepted by the whole box,
        1 = opened internal node, 2 = opened bucket (particles follow)."""
        lo_p, hi_p = box_p[:dim], box_p[dim:]
        th = self.theta * (1.0 - 1e-9)
        fc, nc = t["first_child"], t["n_child"]
        front = np.nonzero(branch)[0]
        out_idx, out_kind = [], []
        while len(front):
            com = t["com"][front]
            v = np.maximum(np.maximum(lo_p - com, com - hi_p), 0.0)
            d = np.sqrt((v * v).sum(axis=1))
            size = 2.0 * t["half"][front]
            acc = (d > 0.0) & (size < th * d)
            isb = fc[front] < 0
            kind = np.where(acc, 0, np.where(isb, 2, 1))
            keep = ~(acc & branch[front])  # accepted branches: the peer has their summary already
            out_idx.append(front[keep])
            out_kind.append(kind[keep])
            op = front[kind == 1]
            cnt = nc[op].astype(np.int64)
            front = np.repeat(fc[op], cnt) + (np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt))
        idx = np.concatenate(out_idx) if out_idx else np.zeros(0, np.int64)
        kind = np.concatenate(out_kind) if out_kind else np.zeros(0, np.int64)
        rows = np.zeros((len(idx), 8 + 2 * dim))
        rows[:, 0] = lvl[idx]
        rows[:, 1] = p1[idx].view(np.float64)
        rows[:, 2] = p2[idx].view(np.float64)
        rows[:, 3] = kind
        rows[:, 4] = t["half"][idx]
        rows[:, 5] = t["mass"][idx]
        rows[:, 6] = np.where(kind == 2, t["pcount"][idx], 0)
        rows[:, 8:8 + dim] = t["center"][idx]
        rows[:, 8 + dim:] = t["com"][idx]
        bsel = idx[kind == 2]
        if len(bsel):  # the opened buckets' particle ranges, concatenated in bucket order
            st = t["pstart"][bsel].astype(np.int64)
            cnt = t["pcount"][bsel].astype(np.int64)
            rel = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            pid = t["pidx"][np.repeat(st, cnt) + rel]
        else:
            pid = np.zeros(0, np.int64)
        parts = np.zeros((len(pid), dim + 2))
        parts[:, :dim] = pos[pid]
        parts[:, dim] = mass[pid]
        parts[:, dim + 1] = gid[pid].astype(np.float64)
        return rows, parts

    def _assemble(self, t, lvl, p1, p2, own_node, pos, mass, gid, top, allbr, rn, rp, dim):
        """One tree in global level order: top nodes, all branches, own
        subtrees, received LET nodes.  Kinds: 0 internal, 1 bucket with
        particles, 2 sealed (a remote node every own bucket accepts)."""
        n = len(gid)
        L_, A_, B_, K_, H_, M_, C_, O_, PC_, SRC_ = [], [], [], [], [], [], [], [], [], []
        # own complete nodes
        if n:
            oi = np.nonzero(own_node)[0]
            L_.append(lvl[oi]); A_.append(p1[oi]); B_.append(p2[oi])
            K_.append(np.where(t["first_child"][oi] < 0, 1, 0))
            H_.append(t["half"][oi]); M_.append(t["mass"][oi]); C_.append(t["center"][oi]); O_.append(t["com"][oi])
            PC_.append(np.where(t["first_child"][oi] < 0, t["pcount"][oi], 0))
            SRC_.append(np.stack([np.zeros(len(oi), np.int64), oi], axis=1))  # (source 0 = own, node)
        # top nodes
        tk = sorted(top)
        if tk:
            L_.append(np.array([L for L, _ in tk], np.int64))
            A_.append(np.array([P >> 63 for _, P in tk], np.uint64))
            B_.append(np.array([P & _M63 for _, P in tk], np.uint64))
            K_.append(np.zeros(len(tk), np.int64))
            H_.append(np.array([top[k][3] for k in tk]))
            M_.append(np.array([top[k][0] for k in tk]))
            C_.append(np.array([top[k][2] for k in tk]).reshape(-1, dim))
            O_.append(np.array([top[k][1] for k in tk]).reshape(-1, dim))
            PC_.append(np.zeros(len(tk), np.int64))
            SRC_.append(np.full((len(tk), 2), -1, np.int64))
        # received LET nodes (kind 0 sealed, 1 internal, 2 bucket) and their particles
        poff = 0
        rpos, rmass, rgid, rsrc = [], [], [], []
        for k, rows in enumerate(rn):
            if not len(rows):
                continue
            kd = rows[:, 3].astype(np.int64)
            L_.append(rows[:, 0].astype(np.int64))
            A_.append(rows[:, 1].copy().view(np.uint64)); B_.append(rows[:, 2].copy().view(np.uint64))
            K_.append(np.where(kd == 0, 2, np.where(kd == 1, 0, 1)))
            H_.append(rows[:, 4]); M_.append(rows[:, 5]); C_.append(rows[:, 8:8 + dim]); O_.append(rows[:, 8 + dim:])
            pc = rows[:, 6].astype(np.int64)
            PC_.append(pc)
            st = np.cumsum(pc) - pc + poff
            SRC_.append(np.stack([np.full(len(rows), 1 + k, np.int64), st], axis=1))
            pr = rp[k]
            rpos.append(pr[:, :dim]); rmass.append(pr[:, dim]); rgid.append(pr[:, dim + 1].astype(np.int64))
            poff += int(pc.sum())
        # remote branches not received: sealed
        for k, br in enumerate(allbr):
            if k == self.comm.rank or not len(br):
                continue
            L_.append(br[:, 0].astype(np.int64))
            A_.append(br[:, 1].copy().view(np.uint64)); B_.append(br[:, 2].copy().view(np.uint64))
            K_.append(np.full(len(br), 3, np.int64))  # 3: branch summary (sealed unless received)
            H_.append(br[:, 3]); M_.append(br[:, 4]); C_.append(br[:, 7:7 + dim]); O_.append(br[:, 7 + dim:])
            PC_.append(np.zeros(len(br), np.int64))
            SRC_.append(np.full((len(br), 2), -1, np.int64))
        lvl_a = np.concatenate(L_); pa = np.concatenate(A_); pb = np.concatenate(B_)
        kind = np.concatenate(K_); half = np.concatenate(H_); nmass = np.concatenate(M_)
        center = np.concatenate(C_).reshape(-1, dim); com = np.concatenate(O_).reshape(-1, dim)
        pcount = np.concatenate(PC_); src = np.concatenate(SRC_)
        # dedupe (level, prefix): a received node overrides a branch summary (kind 3)
        o = _lexsort((kind == 3, pb, pa, lvl_a))
        key = _key16(lvl_a[o], pa[o], pb[o])
        first = np.ones(len(o), bool)
        first[1:] = key[1:] != key[:-1]
        o = o[first]
        key = key[first]
        lvl_a, pa, pb, kind, half, nmass, center, com, pcount, src = _take(
            o, lvl_a, pa, pb, kind, half, nmass, center, com, pcount, src)
        kind[kind == 3] = 2
        nn = len(o)
        # children: nodes of level L + 1 grouped by parent prefix (contiguous, octant order)
        first_child = np.full(nn, -1, np.int64)
        n_child = np.zeros(nn, np.int32)
        has_par = lvl_a > 0
        ci = np.nonzero(has_par)[0]
        pl = lvl_a[ci] - 1
        m1 = np.array([_MASKS[L] >> 63 for L in range(NLEV_MAX + 1)], np.uint64)
        m2 = np.array([_MASKS[L] & _M63 for L in range(NLEV_MAX + 1)], np.uint64)
        pk = _key16(pl, pa[ci] & m1[pl], pb[ci] & m2[pl])
        par = np.searchsorted(key, pk)
        assert np.all(key[np.minimum(par, nn - 1)] == pk), "assembled tree: a node without its parent"
        # children of one parent are contiguous in this order (level, prefix), ci ascending
        n_child = np.bincount(par, minlength=nn).astype(np.int32)
        first_child = np.full(nn, -1, np.int64)
        if len(ci):
            head = np.ones(len(ci), bool)
            head[1:] = par[1:] != par[:-1]
            first_child[par[head]] = ci[head]
        # sealed / bucket nodes must be childless; internal nodes must have children
        assert np.all(n_child[kind != 0] == 0) and np.all(n_child[kind == 0] > 0), "assembled tree: bad node kinds"
        # particles: own, received, one poison row per sealed node (every row
        # appears once in the bucket layout)
        nseal = int(np.sum(kind == 2))
        ppos = [pos] + rpos + [np.full((nseal, dim), np.nan)]
        pmass = [mass] + rmass + [np.zeros(nseal)]
        pgid = [gid] + rgid + [np.full(nseal, -1, np.int64)]
        ppos = np.concatenate(ppos); pmass = np.concatenate(pmass); pgid = np.concatenate(pgid)
        poison = len(pmass) - nseal
        # buckets (kinds 1, 2) in DFS order = order of their left-aligned prefixes
        leaf = np.nonzero(kind != 0)[0]
        leaf = leaf[_lexsort((pb[leaf], pa[leaf]))]
        own_leaf = (kind[leaf] == 1) & (src[leaf, 0] == 0)
        ol = np.nonzero(own_leaf)[0]
        own_lo, own_hi = (int(ol[0]), int(ol[-1]) + 1) if len(ol) else (None, None)
        assert own_lo is not None and own_hi - own_lo == len(ol), "own buckets are not contiguous in DFS order"
        cnt = np.where(kind[leaf] == 2, 1, pcount[leaf]).astype(np.int64)
        cnt[own_leaf] = t["pcount"][src[leaf[own_leaf], 1]]
        # source row of each leaf's first particle: sealed -> its own poison row,
        # received -> n + offset; own leaves take the local DFS particle layout
        seal_rank = np.cumsum(kind[leaf] == 2) - 1
        first = np.where(kind[leaf] == 2, poison + seal_rank, n + np.maximum(src[leaf, 1], 0))
        off = np.concatenate([[0], np.cumsum(cnt)])
        tot = int(off[-1])
        order = np.repeat(first, cnt) + (np.arange(tot) - np.repeat(off[:-1], cnt))
        order[off[own_lo]: off[own_hi]] = t["pidx"]  # own buckets, local DFS order (ascending global id per bucket)
        pstart = np.zeros(nn, np.int64)
        pc_out = np.zeros(nn, np.int64)
        pstart[leaf] = off[:-1]
        pc_out[leaf] = cnt
        assert len(order) == len(pmass) and np.array_equal(np.sort(order), np.arange(len(pmass)))
        tree = dict(center=center, half=half, mass=nmass, com=com, first_child=first_child, n_child=n_child,
                    pstart=pstart, pcount=pc_out, buckets=leaf, order=order, pos=ppos, pmass=pmass, gid=pgid,
                    level=lvl_a, p1=pa, p2=pb, box=self.box, bucket=self.bucket)
        own = (own_lo, own_hi)
        stats = dict(nodes=nn, let_nodes_received=int(sum(len(r) for r in rn)),
                     let_particles_received=int(sum(len(p) for p in rp)), own_buckets=own[1] - own[0])
        return tree, own, stats


def lists_by_prefix(tree: dict, lists, buckets_range):
    """Interaction lists of DFS buckets [b0, b1) of a tree as (level, prefix, kind)
    triples -- comparable across differently numbered trees."""
    ptr, ids, kind = lists[0], lists[1], lists[2]
    b0, b1 = buckets_range
    s = slice(int(ptr[b0]), int(ptr[b1]))
    i = ids[s]
    return (tree["level"][i], tree["p1"][i], tree["p2"][i], kind[s], np.diff(ptr[b0:b1 + 1]))
