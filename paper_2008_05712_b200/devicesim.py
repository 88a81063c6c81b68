"""Occupancy model feeding the combining trigger (mirrors hr/devicesim.py:19-144).

``DeviceSpec`` / ``KernelSpec`` / ``calc_occupancy`` / ``occupancy_oracle``
keep the reference's semantics.  On B200 the specs are not presets: they are
read from the device (``cudaGetDeviceProperties``) and from the real sm_100a
kernels (``cudaFuncGetAttributes``) through ``gc_device_spec`` /
``gc_kernel_spec``.  The simulated cost functions (sim_*) are out of scope:
real CUDA-event timings replace them.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import KernelFitError


@dataclass(frozen=True)
class DeviceSpec:
    sm_count: int
    max_threads_per_sm: int
    max_blocks_per_sm: int
    registers_per_sm: int
    shared_mem_per_sm: int


@dataclass(frozen=True)
class KernelSpec:
    kernel_class: str
    threads_per_block: int
    registers_per_thread: int
    shared_mem_per_block: int
    compute_per_item: float = 0.0
    block_shape: tuple = (0, 0)
    members_per_block: int = 1  # work requests one block serves (warp-per-request kernels: warps/block)


DEVICE_PRESETS = {
    "kepler-k20": DeviceSpec(13, 2048, 16, 65536, 49152),
    "unit": DeviceSpec(1, 128, 1, 65536, 49152),
}

KERNEL_PRESETS = {
    "force": KernelSpec("force", 128, 64, 4096, 0.03, (16, 8)),
    "ewald": KernelSpec("ewald", 128, 100, 6144, 0.02, (16, 8)),
    "md": KernelSpec("md", 128, 64, 4096, 0.002, (16, 8)),
}


def calc_occupancy(k: KernelSpec, d: DeviceSpec):
    """Blocks per SM under the four resource limits (hr/devicesim.py:111-130)."""
    lim = [d.max_blocks_per_sm, d.max_threads_per_sm // k.threads_per_block]
    if k.registers_per_thread > 0:
        lim.append(d.registers_per_sm // (k.registers_per_thread * k.threads_per_block))
    if k.shared_mem_per_block > 0:
        lim.append(d.shared_mem_per_sm // k.shared_mem_per_block)
    blocks = min(lim)
    if blocks <= 0:
        raise KernelFitError(f"kernel {k.kernel_class!r} fits zero blocks per SM (limits {lim})")
    return blocks, blocks * k.threads_per_block / d.max_threads_per_sm


def occupancy_oracle(k: KernelSpec, d: DeviceSpec) -> int:
    """Largest feasible block count by exhaustive search (test oracle)."""
    best = 0
    for b in range(1, d.max_blocks_per_sm + 1):
        if (b * k.threads_per_block <= d.max_threads_per_sm
                and b * k.registers_per_thread * k.threads_per_block <= d.registers_per_sm
                and b * k.shared_mem_per_block <= d.shared_mem_per_sm):
            best = b
    return best


def b200_device_spec(ctx=None) -> DeviceSpec:
    """DeviceSpec of the visible GPU (gc_device_spec)."""
    from . import _lib as L
    v = (ctx or L.context()).device_spec()
    return DeviceSpec(int(v[0]), int(v[1]), int(v[2]), int(v[3]), int(v[4]))


def b200_kernel_spec(kernel_class: str, ctx=None) -> KernelSpec:
    """KernelSpec of a real sm_100a kernel: "force" (BH group force), "walk",
    "force_member" (one warp per work request), "force_slot" (the data-manager
    member kernel gc_bh_run_members launches), "ewald_member", "md" (cell kernel)."""
    from . import _lib as L
    v = (ctx or L.context()).kernel_spec(kernel_class)
    return KernelSpec(kernel_class, int(v[0]), int(v[1]), int(v[2]), members_per_block=int(v[3]))
