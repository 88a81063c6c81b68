"""ctypes binding of libgcharm.so (include/gcharm.h).

There is no fallback: if the CUDA library is missing or no sm_100 device is
visible, every entry point raises.  Build with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``make -C paper_2008_05712_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import CudaError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GCHARM_LIB") or os.path.join(_HERE, "libgcharm.so")  # override: kernel A/B experiments

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
i8p = C.POINTER(C.c_int8)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

# name -> (argtypes); every function returns gc_status (int32) unless listed in _RESTYPE
SIGNATURES = {
    "gc_ctx_create": [C.c_int, C.POINTER(vp)],
    "gc_ctx_destroy": [vp],
    "gc_ctx_sync": [vp],
    "gc_ctx_stream": [vp],
    "gc_device_spec": [vp, i64p],
    "gc_kernel_spec": [vp, C.c_char_p, i64p],
    "gc_forces_from_points": [vp, C.c_int64, C.c_int64, C.c_int32, f64p, f64p, f64p, f64p, C.c_double,
                              C.c_double, f64p],
    "gc_direct_forces": [vp, C.c_int64, C.c_int32, f64p, f64p, C.c_double, C.c_double, f64p],
    "gc_md_cross_forces": [vp, C.c_int64, C.c_int64, C.c_int32, f64p, f64p, C.c_double, C.c_double, f64p, f64p],
    "gc_md_self_forces": [vp, C.c_int64, C.c_int32, f64p, C.c_double, C.c_double, f64p],
    "gc_count_address_runs": [vp, i64p, C.c_int64, C.c_int64, i64p],
    "gc_mdloop_create": [vp, C.POINTER(vp)],
    "gc_mdloop_destroy": [vp],
    "gc_mdloop_set": [vp, C.c_int64, f64p, f64p, i64p, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                      C.c_int32],
    "gc_mdloop_run": [vp, C.c_int32, C.c_double, i64p],
    "gc_mdloop_get_state": [vp, f64p, f64p, i64p],
    "gc_mdloop_topology": [vp, i64p],
    "gc_mdloop_elapsed": [vp, f64p],
    "gc_mdloop_phases": [vp, f64p],
    "gc_ewald_moments": [vp, C.c_int64, f64p, f64p, f64p],
    "gc_ewald_correction": [vp, C.c_int64, f64p, f64p, f64p, f64p, f64p],
    "gc_bh_ewald_moments": [vp, f64p],
    "gc_bh_run_ewald": [vp, vp, i64p, C.c_int32, f64p, C.c_double],
    "gc_bh_get_ewald": [vp, f64p, f64p],
    "gc_bh_create": [vp, C.POINTER(vp)],
    "gc_bh_destroy": [vp],
    "gc_bh_set_particles": [vp, C.c_int64, C.c_int32, f64p, f64p, C.c_double, C.c_int64],
    "gc_bh_sizes": [vp, i64p],
    "gc_bh_set_periodic": [vp, C.c_int32, C.c_double],
    "gc_bh_set_force_mode": [vp, C.c_int32],
    "gc_bh_set_overlap": [vp, C.c_int32],
    "gc_bh_keys": [vp, C.c_int64, C.c_int32, f64p, C.c_double, u64p, u64p],
    "gc_bh_set_forced_splits": [vp, C.c_int64, i32p, u64p],
    "gc_bh_set_tree": [vp, C.c_int64, C.c_int32, C.c_double, C.c_int64, f64p, f64p, f64p, f64p, i64p, i32p, i64p,
                       i64p, C.c_int64, i64p, C.c_int64, i64p, f64p, f64p, C.c_int64, i64p],
    "gc_bh_walk_forces_async": [vp, C.c_double, C.c_double, C.c_double],
    "gc_bh_pair_stats": [vp, i64p],
    "gc_debug_walk_prof": [i64p, C.c_int32],
    "gc_bh_get_tree": [vp, f64p, f64p, f64p, f64p, i64p, i32p, i64p, i64p, i64p],
    "gc_bh_walk": [vp, C.c_double],
    "gc_bh_get_lists": [vp, i64p, i64p, i8p, i64p],
    "gc_bh_set_lists": [vp, C.c_int64, i64p, i64p, i8p],
    "gc_bh_forces": [vp, C.c_double, C.c_double, f64p],
    "gc_bh_forces_async": [vp, C.c_double, C.c_double],
    "gc_bh_forces_potential": [vp, C.c_double, C.c_double, f64p, f64p],
    "gc_bh_interactions": [vp, i64p],
    "gc_bh_timings": [vp, f64p],
    "gc_bh_io_bytes": [vp, i64p, C.c_int32],
    "gc_bh_groups": [vp, i64p, i64p],
    "gc_bh_bucket_work": [vp, i64p],
    "gc_bh_set_range": [vp, C.c_int64, C.c_int64],
    "gc_measure_fp32_peak": [vp, f64p, f64p],
    "gc_bh_step": [vp, C.c_int64, C.c_int32, f64p, f64p, C.c_double, C.c_int64, C.c_double, C.c_double,
                   C.c_double, f64p],
    "gc_md_columns": [vp, i64p],
    "gc_md_forces_columns": [vp, vp, C.c_int64],
    "gc_md_get_forces": [vp, f64p, f64p],
    "gc_md_pack_dev": [vp, C.c_int32, vp, C.c_int64, vp],
    "gc_md_set_ghosts_dev": [vp, vp, vp, vp, vp, C.c_int64],
    "gc_md_slab_step_dev": [vp, C.c_double],
    "gc_md_migrate_dev": [vp, vp, vp, vp, vp, C.c_int64],
    "gc_md_slab_counts": [vp, i64p],
    "gc_batcher_create": [vp, vp, vp, C.c_int64, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(vp)],
    "gc_batcher_destroy": [vp],
    "gc_batcher_submit": [vp, C.c_int64, i64p, f64p, i64p, i64p, i8p],
    "gc_batcher_prepare": [vp, C.c_int64, i64p, C.c_int64],
    "gc_batcher_submit_walk": [vp, C.c_int64, i64p, f64p],
    "gc_batcher_poll": [vp, C.c_double],
    "gc_batcher_flush": [vp, C.c_double],
    "gc_batcher_sync": [vp, i64p],
    "gc_batcher_log": [vp, i64p, f64p],
    "gc_batcher_trigger_device": [C.c_int64, C.c_double, C.c_int32, C.c_int64, f64p, i8p, i64p, i64p, f64p, i64p],
    "gc_dm_create": [vp, C.c_int64, C.c_int64, C.c_int32, C.POINTER(vp)],
    "gc_dm_destroy": [vp],
    "gc_dm_build_plan": [vp, i64p, i64p, C.c_int32, C.c_double, i64p, i64p],
    "gc_dm_plan_get": [vp, i64p, i64p, i64p, i64p],
    "gc_dm_release": [vp, i64p, C.c_int64],
    "gc_dm_pin": [vp, i64p, C.c_int64, C.c_int32],
    "gc_dm_evict": [vp, C.c_int64, i64p, i64p],
    "gc_dm_lookup": [vp, i64p, C.c_int64, C.c_double, i8p],
    "gc_dm_state": [vp, i64p],
    "gc_dm_observe": [vp, i64p, C.c_int64],
    "gc_dm_sorted_index": [vp, i64p, i64p],
    "gc_dm_table": [vp, i64p, i64p, f64p, i64p],
    "gc_md_create": [vp, C.POINTER(vp)],
    "gc_md_destroy": [vp],
    "gc_md_set_system": [vp, C.c_int64, C.c_int32, f64p, f64p, i64p, i64p, C.c_double, C.c_int32, C.c_int32,
                         f64p],
    "gc_md_forces": [vp, f64p, f64p],
    "gc_md_run": [vp, C.c_int32, C.c_double],
    "gc_md_get_state": [vp, f64p, f64p, i64p],
    "gc_md_elapsed": [vp, f64p],
    "gc_dm_stage_bh": [vp, vp],
    "gc_bh_run_members": [vp, vp, i64p, C.c_int32, i8p, C.c_int64, C.c_double, C.c_double],
    "gc_bh_get_forces": [vp, f64p],
    "gc_md_set_slab": [vp, C.c_int64, C.c_int64, i64p],
    "gc_md_pack": [vp, C.c_int32, vp, C.c_int64, i64p],
    "gc_md_set_ghosts": [vp, vp, C.c_int64, vp, C.c_int64],
    "gc_md_slab_step": [vp, C.c_double],
    "gc_md_migrate": [vp, vp, C.c_int64, vp, C.c_int64],
    "gc_md_owned": [vp, i64p, f64p, f64p, i64p],
}
_RESTYPE = {"gc_ctx_stream": vp, "gc_last_error": C.c_char_p, "gc_version": C.c_char_p}

_lib = None
_lock = threading.Lock()


def load():
    """Load libgcharm.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaError(f"{LIB_PATH} is missing: build the CUDA extension first (__graft_entry__.build())")
            L = C.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, C.c_int32)
            for name, rt in _RESTYPE.items():
                getattr(L, name).restype = rt
            L.gc_last_error.argtypes = []
            L.gc_version.argtypes = []
            _lib = L
    return _lib


def call(name, *args):
    L = load()
    st = getattr(L, name)(*args)
    if st:
        raise_for_status(st, f"{name}: {L.gc_last_error().decode(errors='replace')}")


class Context:
    """One CUDA device + stream owned by libgcharm (gc_ctx)."""

    def __init__(self, device: int = 0):
        self.handle = vp()
        call("gc_ctx_create", int(device), C.byref(self.handle))
        self.device = device

    @property
    def stream(self) -> int:
        return load().gc_ctx_stream(self.handle)

    def sync(self):
        call("gc_ctx_sync", self.handle)

    def device_spec(self):
        out = np.zeros(6, np.int64)
        call("gc_device_spec", self.handle, ptr(out, i64p))
        return out

    def kernel_spec(self, kernel_class: str):
        out = np.zeros(5, np.int64)
        call("gc_kernel_spec", self.handle, kernel_class.encode(), ptr(out, i64p))
        return out

    def __del__(self):
        try:
            if self.handle:
                load().gc_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("GCHARM_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _lock:
        c = _ctx.get(device)
    if c is None:
        c = Context(device)
        with _lock:
            _ctx[device] = c
    return c


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)
