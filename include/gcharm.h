/*
 * gcharm.h -- C ABI of libgcharm.so, the B200 (sm_100a) drop-in for the
 * G-Charm irregular force path of hetero-rt (arXiv 2008.05712 reference).
 *
 * Plain C types only: pointers, sizes, doubles.  Every call returns a
 * gc_status (0 = ok); gc_last_error() gives the message of the last failure on
 * the calling thread.  Status codes map 1:1 onto the reference's exception
 * classes (hr/errors.py:4-53):
 *
 *   GC_E_CAPACITY  -> CapacityError   (hr/errors.py:32)
 *   GC_E_GROUPING  -> GroupingError   (hr/errors.py:24)
 *   GC_E_CLOCK     -> ClockError      (hr/errors.py:20)
 *   GC_E_KERNELFIT -> KernelFitError  (hr/errors.py:28)
 *   GC_E_VALUE     -> ValueError      (e.g. bucket_size < 1, nbody.py:80)
 *   GC_E_CUDA / GC_E_NOMEM -> HeteroRtError (hr/errors.py:4)
 *
 * Ownership: inputs are caller-owned and read only; outputs are
 * caller-allocated.  Device state (trees, lists, slot pools, reuse tables)
 * is owned by the handle that created it.  One host thread per handle; each
 * context owns one CUDA stream.  Calls that take host buffers synchronise
 * before returning; *_async calls only enqueue on the context stream.
 */
#ifndef GCHARM_H
#define GCHARM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gc_status;
enum {
    GC_OK = 0,
    GC_E_VALUE = 1,
    GC_E_CAPACITY = 2,
    GC_E_GROUPING = 3,
    GC_E_CLOCK = 4,
    GC_E_KERNELFIT = 5,
    GC_E_CUDA = 6,
    GC_E_NOMEM = 7,
    GC_E_STATE = 8
};

typedef struct gc_ctx gc_ctx;
typedef struct gc_bh gc_bh;
typedef struct gc_dm gc_dm;
typedef struct gc_md gc_md;
typedef struct gc_batcher gc_batcher;

const char *gc_last_error(void);
const char *gc_version(void);

/* ---- context ------------------------------------------------------------ */
gc_status gc_ctx_create(int device, gc_ctx **out);
gc_status gc_ctx_destroy(gc_ctx *ctx);
gc_status gc_ctx_sync(gc_ctx *ctx);
/* the context's cudaStream_t, for event timing by the caller */
void *gc_ctx_stream(gc_ctx *ctx);

/* Device limits for the occupancy model (replaces DeviceSpec presets,
 * hr/devicesim.py:19-27,63-78): out[0..5] = sm_count, max_threads_per_sm,
 * max_blocks_per_sm, registers_per_sm, shared_mem_per_sm, clock_khz. */
gc_status gc_device_spec(gc_ctx *ctx, int64_t out[6]);

/* Kernel resources of a real kernel class (replaces KernelSpec presets,
 * hr/devicesim.py:30-39,83-108): out[0..4] = threads_per_block,
 * registers_per_thread, shared_mem_per_block, members_per_block,
 * cuda_occupancy_blocks_per_sm.  kernel_class: "force", "md", "walk". */
gc_status gc_kernel_spec(gc_ctx *ctx, const char *kernel_class, int64_t out[5]);

/* FP32 FFMA throughput probe (roofline denominator): TFLOP/s and ms */
gc_status gc_measure_fp32_peak(gc_ctx *ctx, double *tflops, double *ms);

/* ---- hr/kernels.py entry points (host buffers, float64 in/out) ------------ */
/* forces_from_points (hr/kernels.py:70-98) */
gc_status gc_forces_from_points(gc_ctx *ctx, int64_t n, int64_t m, int32_t dim, const double *ppos,
                                const double *pmass, const double *spos, const double *smass, double g,
                                double eps, double *out);
/* direct_forces (hr/kernels.py:40-63) */
gc_status gc_direct_forces(gc_ctx *ctx, int64_t n, int32_t dim, const double *pos, const double *mass,
                           double g, double eps, double *out);
/* md_cross_forces (hr/kernels.py:105-135): fa (na x dim), fb (nb x dim) */
gc_status gc_md_cross_forces(gc_ctx *ctx, int64_t na, int64_t nb, int32_t dim, const double *pa,
                             const double *pb, double cutoff, double stiffness, double *fa, double *fb);
/* md_self_forces (hr/kernels.py:138-161) */
gc_status gc_md_self_forces(gc_ctx *ctx, int64_t n, int32_t dim, const double *p, double cutoff,
                            double stiffness, double *out);
/* count_address_runs (hr/kernels.py:213-216) */
gc_status gc_count_address_runs(gc_ctx *ctx, const int64_t *addresses, int64_t n, int64_t group,
                                int64_t *out);

/* ---- Barnes-Hut bucket forces (hr/workloads/nbody.py) ---------------------- */
gc_status gc_bh_create(gc_ctx *ctx, gc_bh **out);
gc_status gc_bh_destroy(gc_bh *bh);
/* Particles (host, float64, float32-representable) + tree build.
 * Restates build_bucket_tree (nbody.py:78-135): level-order node ids, DFS
 * bucket order, float64 mass/COM with the reference's rounding sequence. */
gc_status gc_bh_set_particles(gc_bh *bh, int64_t n, int32_t dim, const double *pos, const double *mass,
                              double box, int64_t bucket_size);
/* Tree build on the GPU (device != 0, the default) or the host C++ build;
 * both are bit-identical to build_bucket_tree.  Applies to the next
 * gc_bh_set_particles / gc_bh_step. */
/* 1 (default): the reorganisation into per-force-group source runs happens in
 * shared memory inside the force kernel; 0: expand_kernel writes the runs to an
 * HBM staging buffer first (A/B and the HBM roofline of the staging layer).
 * Forces are bit-identical either way. */
gc_status gc_bh_set_force_mode(gc_bh *bh, int32_t fused);
/* walk instrumentation, only in builds with -DWALK_PROF=1 (zeros otherwise):
 * out = node visits, sum of active buckets, visits with an empty half, decisions,
 * ns from the first warp's start to the first warp without work, to the last warp's exit */
gc_status gc_debug_walk_prof(int64_t out[6], int32_t reset);
/* pairs the force kernel evaluates for the current lists: out[0] = padded
 * source records x 32 lanes summed over force groups, out[1] = padded records
 * x targets; useful pairs = gc_bh_interactions (full walk-group range) */
gc_status gc_bh_pair_stats(gc_bh *bh, int64_t out[2]);
/* 1: gc_bh_walk_forces_async / gc_bh_step run the walk and the fused force
 * kernel concurrently (force groups consumed as their walk groups finish);
 * the force kernel is a programmatic dependent launch that starts when every
 * walk block has a warp out of work.  2: one persistent kernel does both
 * (walk_force_kernel: a warp drains walk items, then force groups from the
 * readiness queue; its shared memory holds either the walk stack or the
 * force ring).  Results are identical in all modes.  Default 0 (1 and 2
 * measured neutral / slower); timings then report the whole step as the walk. */
gc_status gc_bh_set_overlap(gc_bh *bh, int32_t on);

/* --- Distributed Barnes-Hut (paper_2008_05712_b200/bh_dist.py) ---
 * The reference has no distributed path: it runs one process
 * (hr/workloads/nbody.py:78-250).  These entry points let each rank build the
 * part of the GLOBAL tree it owns and walk its own buckets over an assembled
 * locally-essential tree, with lists bit-identical to the one-GPU tree.
 *
 * Octant keys of the device build (nbody.py:97-108 descent, 3 bits per level,
 * levels 0-20 in k1, 21-41 in k2; digits of levels with half < 1e-9 are 0). */
gc_status gc_bh_keys(gc_ctx *ctx, int64_t n, int32_t dim, const double *pos, double box, uint64_t *k1,
                     uint64_t *k2);
/* Cubes (level, key prefix of levels < level as (k1, k2)) that the next device
 * build splits whatever their local particle count -- they straddle ranks and
 * hold more than bucket_size particles globally.  n = 0 clears the list. */
gc_status gc_bh_set_forced_splits(gc_bh *bh, int64_t n, const int32_t *level, const uint64_t *prefix /* 2n */);
/* Upload an assembled tree in the reference's layout (level-order node ids;
 * first_child = -1 for buckets; buckets in depth-first order; order = particle
 * ids of the buckets' ranges into pos / pmass).  Walk groups never straddle
 * the DFS bucket indices `cuts` (a rank's own buckets form whole groups, then
 * gc_bh_set_range selects them). */
gc_status gc_bh_set_tree(gc_bh *bh, int64_t n_nodes, int32_t dim, double box, int64_t bucket_size,
                         const double *center, const double *half, const double *mass, const double *com,
                         const int64_t *first_child, const int32_t *n_child, const int64_t *pstart,
                         const int64_t *pcount, int64_t n_buckets, const int64_t *buckets, int64_t n_parts,
                         const int64_t *order, const double *pos, const double *pmass, int64_t n_cuts,
                         const int64_t *cuts);
/* one step's walk + forces, asynchronous (= gc_bh_walk + gc_bh_forces_async) */
gc_status gc_bh_walk_forces_async(gc_bh *bh, double theta, double g, double eps);
/* Sizes: out[0..4] = n_nodes, n_buckets, per-bucket list entries, union
 * entries of the last device walk, source records they expand to (staging) */
/* Periodic Barnes-Hut (no reference implementation, the
 * float64 restatement is oracle/gcharm_oracle.c orc_periodic_forces): with
 * nrep > 0 every bucket walks the tree once per image of the box (side L =
 * the tree's box, (2 nrep + 1)^3 images, node centres of mass shifted in the
 * opening test; nrep <= 1: ChaNGa's nReplicas) and the fused force kernel
 * evaluates the shifted sources.
 * Per-bucket counts (gc_bh_get_lists ptr / item_count) cover all images; the
 * per-bucket id lists, potentials, the staged mode and the overlap are
 * unavailable.  nrep = 0 restores the open-boundary walk. */
gc_status gc_bh_set_periodic(gc_bh *bh, int32_t nrep, double L);
gc_status gc_bh_sizes(gc_bh *bh, int64_t out[5]);
/* Tree arrays (host, caller-allocated by gc_bh_sizes): any pointer may be NULL */
gc_status gc_bh_get_tree(gc_bh *bh, double *center, double *half, double *mass, double *com,
                         int64_t *first_child, int32_t *n_child, int64_t *pcount, int64_t *buckets,
                         int64_t *pidx);
/* Device opening-angle walk (build_interaction_lists, nbody.py:160-199) with
 * bit-exact float64 decisions; lists stay in HBM. */
gc_status gc_bh_walk(gc_bh *bh, double theta);
/* Lists to host in walk order (CSR over buckets in DFS order):
 * kind 0 = node_interactions, 1 = particle_interactions. */
gc_status gc_bh_get_lists(gc_bh *bh, int64_t *ptr, int64_t *ids, int8_t *kind, int64_t *item_count);
/* Lists from the host runtime (the drop-in path when the walk ran elsewhere) */
gc_status gc_bh_set_lists(gc_bh *bh, int64_t n_buckets, const int64_t *ptr, const int64_t *ids,
                          const int8_t *kind);
/* eval_forces (nbody.py:216-250): float64 out (n x dim), original particle order */
gc_status gc_bh_forces(gc_bh *bh, double g, double eps, double *out);
/* Forces plus per-particle potential energy -G m_i sum_j m_j / sqrt(r^2 + eps^2)
 * over the same interaction lists (pot: n float64).  No reference counterpart
 * (restated next to forces_from_points). */
gc_status gc_bh_forces_potential(gc_bh *bh, double g, double eps, double *out, double *pot);
/* Enqueue only (results stay on device); for device-resident timing */
gc_status gc_bh_forces_async(gc_bh *bh, double g, double eps);
/* Sum over buckets of n_b * item_count_b (the interaction count) */
gc_status gc_bh_interactions(gc_bh *bh, int64_t *out);
/* Device time (ms, CUDA events on the context stream) of the last walk
 * (out[0]), the last force kernel (out[1]) and the reorganisation (staging
 * gather) that precedes it (out[2]). */
gc_status gc_bh_timings(gc_bh *bh, double out[3]);
/* Host<->device bytes moved since the last reset (out[0] = H2D, out[1] = D2H);
 * gc_bh_step resets at entry, so after it these are that step's bytes. */
gc_status gc_bh_io_bytes(gc_bh *bh, int64_t out[2], int32_t reset);
/* Multi-GPU sharding: walk groups (32 consecutive DFS buckets each) and the
 * per-bucket work n_b * item_count_b of the last walk; gc_bh_set_range
 * restricts walk + forces to walk groups [wg_begin, wg_end) (a shard chosen
 * by the K-way generalisation of partition_queue, hr/scheduler.py:73-107). */
gc_status gc_bh_groups(gc_bh *bh, int64_t *n_walk_groups, int64_t *wg_first_bucket /* n+1, may be NULL */);
gc_status gc_bh_bucket_work(gc_bh *bh, int64_t *work /* n_buckets */);
gc_status gc_bh_set_range(gc_bh *bh, int64_t wg_begin, int64_t wg_end);
/* End-to-end step from host buffers: H2D particles, tree, device walk,
 * forces, D2H forces (n x dim float64). */
gc_status gc_bh_step(gc_bh *bh, int64_t n, int32_t dim, const double *pos, const double *mass, double box,
                     int64_t bucket_size, double theta, double g, double eps, double *out);

/* ---- data manager (hr/memory.py:228-369) ------------------------------------
 * One handle per kernel class: uniform slots of slot_bytes over
 * capacity_bytes of HBM, mode 0 = REDUNDANT, 1 = REUSE, 2 = REUSE_SORTED
 * (MemoryMode, memory.py:30-33).  Buffer ids are non-negative int32. */
gc_status gc_dm_create(gc_ctx *ctx, int64_t capacity_bytes, int64_t slot_bytes, int32_t mode, gc_dm **out);
gc_status gc_dm_destroy(gc_dm *dm);
/* build_plan (memory.py:289-360): members as CSR (ids, bounds[n_members+1]).
 * Pins the batch's buffers until gc_dm_release.  GC_E_CAPACITY on failure
 * (pins rolled back).  Sizes of the plan are returned; fetch it with
 * gc_dm_plan_get. */
gc_status gc_dm_build_plan(gc_dm *dm, const int64_t *ids, const int64_t *bounds, int32_t n_members, double now,
                           int64_t *n_transfer, int64_t *n_positions);
/* to_transfer (buffer ids, in allocation order), addresses (slot per
 * position), transactions per member (memory.py:204-209); out_bytes =
 * {total_bytes, indirection_bytes, indirect}.  Any pointer may be NULL. */
gc_status gc_dm_plan_get(gc_dm *dm, int64_t *to_transfer, int64_t *addresses, int64_t *transactions,
                         int64_t out_bytes[3]);
/* release_batch (memory.py:362-365): unpin set(ids) */
gc_status gc_dm_release(gc_dm *dm, const int64_t *ids, int64_t n);
/* pin / unpin set(ids) (memory.py:240-250): delta +1 or -1 */
gc_status gc_dm_pin(gc_dm *dm, const int64_t *ids, int64_t n, int32_t delta);
/* evict_slots (memory.py:260-285): evicted buffer ids in eviction order */
gc_status gc_dm_evict(gc_dm *dm, int64_t needed_bytes, int64_t *evicted, int64_t *n_evicted);
/* lookup_residency (memory.py:78-93): resident[i] = 1 if ids[i] has a slot
 * (and its last_use_time becomes now) */
gc_status gc_dm_lookup(gc_dm *dm, const int64_t *ids, int64_t n, double now, int8_t *resident);
/* observe_indices (memory.py:252-256) into the SortedIndexArray
 * (memory.py:125-179) held on the device: gc_dm_observe appends ids in order
 * (every call = one insert per id, the reference's binary-insertion
 * comparison count computed exactly from each insertion's set size and rank);
 * gc_dm_sorted_index: out = {size, comparisons, inserts}, indices ascending
 * (may be NULL). */
gc_status gc_dm_observe(gc_dm *dm, const int64_t *ids, int64_t n);
gc_status gc_dm_sorted_index(gc_dm *dm, int64_t out[3], int64_t *indices);
/* out = {slot_count, free_slots, resident_buffers, id_universe} */
gc_status gc_dm_state(gc_dm *dm, int64_t out[4]);
/* resident table sorted by buffer id (ChareTable, memory.py:50-75) */
gc_status gc_dm_table(gc_dm *dm, int64_t *bufs, int64_t *slots, double *last_use, int64_t *pins);

/* ---- combined work requests on the device (replaces the cost model at the
 * GPU launch site, hr/timeline.py:300-321) ----------------------------------
 * gc_dm_stage_bh: copy the last plan's transferred buffers (tree node ids)
 * into their slots -- slot = [com hi, mass][com lo, pcount][bucket particles];
 * the B200 form of the reference's H2D transfer (hr/timeline.py:307-316).
 * gc_bh_run_members: members = DFS bucket indices of the combined request,
 * kinds per plan position (0 node_interaction, 1 particle_interaction) in the
 * plan's position order (per-member id order in REUSE_SORTED); forces of the
 * members' particles into the tree's force array.  gc_bh_get_forces: D2H. */
gc_status gc_dm_stage_bh(gc_dm *dm, gc_bh *bh);
gc_status gc_bh_run_members(gc_bh *bh, gc_dm *dm, const int64_t *member_buckets, int32_t n_members,
                            const int8_t *kinds, int64_t n_positions, double g, double eps);
gc_status gc_bh_get_forces(gc_bh *bh, double *out);

/* ---- device batcher (north star subsystem (1)) ------------
 * The aggregation trigger of hr/aggregator.py (observe_arrival / poll_combine,
 * :41-110; size rule = exactly max_size earliest, timeout rule = strict gap >
 * timeout_factor x running-max gap over the last `window` gaps, 0 = all) over
 * a device ring of work requests, each emitted batch planned by the device
 * data manager `dm` (no host round trip when every buffer id fits the slot
 * count, else the synchronous plan), staged into its slots and evaluated by
 * one member-kernel launch -- the launch site hr/timeline.py:300-321 executes
 * instead of charging its cost model.  One batcher per kernel class.
 * gc_batcher_submit: n requests in FIFO order, owners = DFS bucket indices,
 *   arrival times (non-decreasing; GC_E_CLOCK otherwise), buffer ids as CSR
 *   (ptr[n+1] into ids) with kinds (0 node_interaction, 1
 *   particle_interaction); every arrival is observed and polled at its time
 *   (Runtime.submit_work_request hr/runtime.py:151-163 + _poll_aggregation
 *   hr/timeline.py:262-274), emitted batches are launched asynchronously.
 * gc_batcher_poll: a poll at `now` (Timeline ticks).
 * gc_batcher_flush: end of the phase, drain in max_size chunks
 *   (hr/timeline.py:276-283).
 * gc_batcher_sync: wait for every launched batch; n_batches emitted so far.
 * gc_batcher_log: ScheduleLog rows (hr/timeline.py:63-100), 7 int64 per batch
 *   {combined_id, first request, members, positions, buffers transferred,
 *   transactions, synchronous plan} and 2 doubles {emit time, device ms}.
 * gc_batcher_trigger_device: the trigger alone, evaluated on the device on
 *   n events at the given times (or %globaltimer stamps when arrival is
 *   NULL): an arrival (observed, then polled) or, where is_poll[i] != 0, a
 *   poll only; emissions (first request, count, time). */
gc_status gc_batcher_create(gc_ctx *ctx, gc_bh *bh, gc_dm *dm, int64_t max_size, double timeout_factor,
                            int32_t window, double g, double eps, gc_batcher **out);
gc_status gc_batcher_destroy(gc_batcher *b);
gc_status gc_batcher_submit(gc_batcher *b, int64_t n, const int64_t *owner, const double *arrival,
                            const int64_t *ptr, const int64_t *ids, const int8_t *kinds);
/* gc_batcher_prepare: optional, before a phase of n requests (CSR ptr[n+1],
 * largest buffer id max_id): every device buffer and plan scratch is sized up
 * front so the submission path never allocates. */
gc_status gc_batcher_prepare(gc_batcher *b, int64_t n, const int64_t *ptr, int64_t max_id);
/* gc_batcher_submit_walk: as gc_batcher_submit, every request's buffers
 * being its owner bucket's interaction list as the device walk left it in HBM
 * (requires gc_bh_get_lists with ids on the current walk): no buffer id
 * crosses from the host, only owners and arrival times. */
gc_status gc_batcher_submit_walk(gc_batcher *b, int64_t n, const int64_t *owner, const double *arrival);
gc_status gc_batcher_poll(gc_batcher *b, double now);
gc_status gc_batcher_flush(gc_batcher *b, double now);
gc_status gc_batcher_sync(gc_batcher *b, int64_t *n_batches);
gc_status gc_batcher_log(gc_batcher *b, int64_t *rows, double *times);
gc_status gc_batcher_trigger_device(int64_t max_size, double timeout_factor, int32_t window, int64_t n,
                                    const double *arrival, const int8_t *is_poll, int64_t *e_first, int64_t *e_count, double *e_time,
                                    int64_t *n_emit);

/* ---- cell-pair MD (hr/workloads/md.py; 3-D Lennard-Jones extension) --------
 * law 0: soft repulsion, params = {cutoff, stiffness, -} (kernels.py:105-161);
 * law 1: Lennard-Jones, params = {rc, epsilon, sigma} (no reference; oracle/).
 * dims = cells per dimension (2-D: {rows, cols, 1}); cell_of (optional) is the
 * caller's initial patch assignment (PatchGrid.patch_of, md.py:32).  Periodic
 * grids need >= 3 cells per dimension. */
gc_status gc_md_create(gc_ctx *ctx, gc_md **out);
gc_status gc_md_destroy(gc_md *md);
gc_status gc_md_set_system(gc_md *md, int64_t n, int32_t dim, const double *pos, const double *vel,
                           const int64_t *cell_of, const int64_t dims[3], double cell_size, int32_t periodic,
                           int32_t law, const double params[3]);
/* compute_forces (md.py:121-163) on the current state: forces (n x dim) and,
 * for LJ, per-atom energy (half of each pair energy); either may be NULL */
gc_status gc_md_forces(gc_md *md, double *forces, double *energy);
/* `steps` iterations of md_step (md.py:166-190) on the device (CUDA graph) */
gc_status gc_md_run(gc_md *md, int32_t steps, double dt);
gc_status gc_md_get_state(gc_md *md, double *pos, double *vel, int64_t *cell_of);
/* device time (ms, CUDA events) of the last gc_md_forces, gc_md_run or gc_md_slab_step */
gc_status gc_md_elapsed(gc_md *md, double *ms);

/* ---- x-slab spatial decomposition (multi-GPU MD) -------------
 * The reference has no multi-process MD: the patch loop of compute_forces /
 * md_step (hr/workloads/md.py:121-190) runs in one process.  A slab handle
 * owns global x cells [gx0, gx0 + nx - 2) of a periodic gnx x ny x nz grid;
 * gc_md_set_system is called with the local dims (owned + 2 ghost planes)
 * and the owned atoms (global coordinates).  Per step: pack ghost planes
 * (what 0 = left, 1 = right) -> exchange -> gc_md_set_ghosts ->
 * gc_md_slab_step -> pack migrants (what 2 = left, 3 = right) -> exchange ->
 * gc_md_migrate.  Pointers to packed records are DEVICE pointers (ghost
 * record = double4 (x, y, z, global id bits); migrant = 2 x double4, + (v, 0)).
 * Forces, positions and decisions are bit-identical to the whole-domain run. */
gc_status gc_md_set_slab(gc_md *md, int64_t gx0, int64_t gnx, const int64_t *gid /* host, owned; may be NULL */);
gc_status gc_md_pack(gc_md *md, int32_t what, void *out /* device, may be NULL */, int64_t cap, int64_t *count);
gc_status gc_md_set_ghosts(gc_md *md, const void *left, int64_t n_left, const void *right, int64_t n_right);
gc_status gc_md_slab_step(gc_md *md, double dt);
gc_status gc_md_migrate(gc_md *md, const void *in_left, int64_t n_left, const void *in_right, int64_t n_right);
gc_status gc_md_owned(gc_md *md, int64_t *n_owned, double *pos, double *vel, int64_t *gid /* host; may be NULL */);
/* Column work requests (configs[4]: LJ force work arriving at a varying
 * generation rate, combined by the batcher's trigger): gc_md_columns out =
 * {columns (0 = the column kernel does not apply), home cells per column,
 * columns along z}; column c = (x * ny + y) * (columns along z) + z-block.
 * gc_md_forces_columns launches the forces of the home cells of a DEVICE
 * int32 column list (asynchronous; positions as last sorted); gc_md_get_forces
 * downloads the force array as it stands. */
gc_status gc_md_columns(gc_md *md, int64_t out[3]);
gc_status gc_md_forces_columns(gc_md *md, const int32_t *cols, int64_t n);
gc_status gc_md_get_forces(gc_md *md, double *forces, double *energy);

/* Device-count slab path (no host round trip inside a step; §8e): the same
 * step with every count on the device.  gc_md_pack_dev writes the records of
 * `what` into a fixed-capacity DEVICE buffer and their number into the DEVICE
 * int32 *count (records beyond cap are dropped and flagged); the *_dev
 * receivers read the received counts from DEVICE int32 pointers.  Exchange
 * the buffers and counts by stream-ordered peer sends (NCCL) on the context's
 * stream.  gc_md_slab_counts synchronises: out = {owned, owned + ghosts,
 * overflow flags (1 message, 2 atom capacity)}; gc_md_owned checks them. */
gc_status gc_md_pack_dev(gc_md *md, int32_t what, void *out, int64_t cap, int32_t *count);
gc_status gc_md_set_ghosts_dev(gc_md *md, const void *left, const int32_t *n_left, const void *right,
                               const int32_t *n_right, int64_t cap);
gc_status gc_md_slab_step_dev(gc_md *md, double dt);
gc_status gc_md_migrate_dev(gc_md *md, const void *in_left, const int32_t *n_left, const void *in_right,
                            const int32_t *n_right, int64_t cap);
gc_status gc_md_slab_counts(gc_md *md, int64_t out[3]);

/* ---- closed-loop MD ----------------------------------------
 * hr/workloads/md.py MDWorkload (md.py:209-271) run on the device as one
 * persistent kernel: per step, patch "interact" messages complete pair
 * entries through readiness counters (hr/runtime.py:95-118), completed
 * entries enqueue their work request, blocks execute requests as they become
 * ready, and the completion count is the step barrier that triggers md_step
 * (md.py:166-190).  Float64, bit-identical to the reference's numba kernels. */
typedef struct gc_mdloop gc_mdloop;
gc_status gc_mdloop_create(gc_ctx *ctx, gc_mdloop **out);
gc_status gc_mdloop_destroy(gc_mdloop *loop);
/* PatchGrid (md.py:29-50): pos/vel (n x 2), patch_of (n); MDParams cutoff / stiffness / periodic */
gc_status gc_mdloop_set(gc_mdloop *loop, int64_t n, const double *pos, const double *vel, const int64_t *patch_of,
                        int32_t rows, int32_t cols, double patch_size, double cutoff, double stiffness,
                        int32_t periodic);
/* `steps` step barriers = steps - 1 md_step updates (MDParams.steps, md.py:263-271);
 * stats (optional, steps x 4): work requests, interact messages, completions, barrier fired */
gc_status gc_mdloop_run(gc_mdloop *loop, int32_t steps, double dt, int64_t *stats);
gc_status gc_mdloop_get_state(gc_mdloop *loop, double *pos, double *vel, int64_t *patch_of);
/* out[3]: patches, pair chares (neighbor_pairs), compute_forces segments */
gc_status gc_mdloop_topology(gc_mdloop *loop, int64_t out[3]);
gc_status gc_mdloop_elapsed(gc_mdloop *loop, double *ms);
/* per step of the last run (steps x 5, ns): counts + scans, scatter, patch
 * sort / gather / messages, execution + barrier, md_step + resets */
gc_status gc_mdloop_phases(gc_mdloop *loop, double *out);

/* ---- Ewald kernel class ------------------------------------
 * The reference models an "ewald" class (one request per bucket, buffers
 * [bucket], item_count max(1, n_b): hr/workloads/nbody.py:317-323; cost
 * hr/devicesim.py:92-99) without computing it.  Here it is the periodic
 * correction of each particle from the root multipole, Hernquist-Bouchet-Suto
 * Ewald summation, float64.  moments[10] = M, com(3), traceless quadrupole
 * Q xx yy zz xy xz yz; params[5] = box L, alpha (<= 0: 2/L), nrep, ewcut, hcut.
 * acc: correction acceleration per unit mass (G = 1); pot: potential. */
gc_status gc_ewald_moments(gc_ctx *ctx, int64_t n, const double *pos, const double *mass, double moments[10]);
gc_status gc_ewald_correction(gc_ctx *ctx, int64_t n, const double *pos, const double moments[10],
                              const double params[5], double *acc, double *pot);
gc_status gc_bh_ewald_moments(gc_bh *bh, double moments[10]);
/* one combined "ewald" request: members = DFS buckets, one buffer each (the
 * last gc_dm plan), payloads staged by gc_dm_stage_bh; forces g m_i a_i */
gc_status gc_bh_run_ewald(gc_bh *bh, gc_dm *dm, const int64_t *member_buckets, int32_t n_members,
                          const double params[5], double g);
gc_status gc_bh_get_ewald(gc_bh *bh, double *forces /* n x 3 */, double *pot /* n; may be NULL */);

#ifdef __cplusplus
}
#endif
#endif /* GCHARM_H */
