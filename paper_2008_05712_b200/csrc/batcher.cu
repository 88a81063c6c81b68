// batcher.cu -- the device batcher (north star subsystem (1)).
//
// The reference combines work requests with a host-side trigger
// (observe_arrival / poll_combine, hr/aggregator.py:41-110, polled after every
// event by Timeline._poll_aggregation, hr/timeline.py:262-274) and then CHARGES
// a cost model for the combined launch (Timeline._launch_gpu,
// hr/timeline.py:300-321).  Here a whole stream of work requests is handed in
// at once (vectorised submission: owners, arrival times and the buffer CSR);
// its buffer ids stay resident in a device ring, the trigger restates
// poll_combine exactly (size rule: exactly max_size earliest; timeout rule:
// strict gap > factor x running-max gap, windowed max optional), and every
// emitted batch -- a contiguous FIFO range of the ring -- is planned by the
// device data manager (residency / LRU / min-free-slot / per-member address
// maps, no host round trip: dm_plan_async), staged into its slots and
// evaluated by one member-kernel launch, all enqueued asynchronously.  The
// host synchronises once (gc_batcher_sync) and reads the ScheduleLog rows
// (hr/timeline.py:63-100) with real device times.
//
// The trigger is one __host__ __device__ function: the parity mode evaluates
// it on the host as the requests are submitted (arrival times given), the
// real-time mode (gc_batcher_trigger_device) evaluates it in a device kernel
// on %globaltimer arrival stamps.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "dm_state.h"

namespace gc {

constexpr int TRIG_WMAX = 256;  // longest arrival-gap window (AggregatorState.window)

// AggregatorState (hr/aggregator.py:27-38) without the request objects: the
// pending FIFO is a count, its requests are the ring's next `npending`.
struct TrigState {
    long long max_size;
    double factor;
    int window;
    int has_interval, has_last;
    double max_interval, last;
    long long npending;
    int gap_head, gap_n;
    double gaps[TRIG_WMAX];
};

// observe_arrival (hr/aggregator.py:41-58); returns 1 on a clock regression (ClockError)
__host__ __device__ inline int trig_observe(TrigState &t, double now)
{
    if (t.has_last) {
        if (now < t.last) return 1;
        const double gap = now - t.last;
        if (t.window > 0) {
            t.gaps[(t.gap_head + t.gap_n) % TRIG_WMAX] = gap;
            if (t.gap_n < t.window) ++t.gap_n;
            else t.gap_head = (t.gap_head + 1) % TRIG_WMAX;
            double m = t.gaps[t.gap_head];
            for (int i = 1; i < t.gap_n; ++i) m = fmax(m, t.gaps[(t.gap_head + i) % TRIG_WMAX]);
            t.max_interval = m;
        } else {
            t.max_interval = t.has_interval ? fmax(t.max_interval, gap) : gap;
        }
        t.has_interval = 1;
    }
    t.last = now;
    t.has_last = 1;
    return 0;
}

// poll_combine (hr/aggregator.py:91-110): requests to take (0: none)
__host__ __device__ inline long long trig_poll(TrigState &t, double now)
{
    if (t.npending == 0) return 0;
    if (t.npending >= t.max_size) {
        t.npending -= t.max_size;
        return t.max_size;
    }
    if (!t.has_interval || !t.has_last) return 0;
    if (now - t.last > t.factor * t.max_interval) {
        const long long k = t.npending;
        t.npending = 0;
        return k;
    }
    return 0;
}

__device__ __forceinline__ double globaltimer_s()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (double)t * 1e-9;
}

// Real-time trigger: n arrivals (device times, or %globaltimer stamps taken
// here when times == nullptr), each observed then polled at its arrival;
// emissions (first request, count, time) in order.  One thread: the trigger is
// a sequential recurrence (running max gap, FIFO).
__global__ void batcher_trigger_kernel(TrigState *st, long long first, int n, const double *__restrict__ times,
                                       const signed char *__restrict__ is_poll, long long *__restrict__ e_first, long long *__restrict__ e_count,
                                       double *__restrict__ e_time, int *__restrict__ n_emit, int *__restrict__ err)
{
    if (threadIdx.x || blockIdx.x) return;
    TrigState t = *st;
    long long head = first - t.npending;  // first pending request
    int ne = 0;
    for (int i = 0; i < n; ++i) {
        const double now = times ? times[i] : globaltimer_s();
        if (!(is_poll && is_poll[i])) {  // an arrival (else a poll only: a timeline tick)
            t.npending += 1;
            if (trig_observe(t, now)) {
                *err = 1;
                break;
            }
        }
        for (long long k; (k = trig_poll(t, now)) > 0;) {
            e_first[ne] = head;
            e_count[ne] = k;
            e_time[ne] = now;
            ++ne;
            head += k;
        }
    }
    *n_emit = ne;
    *st = t;
}

// the device-walk lists of owners[0..n) appended to the ring: request k's
// positions [ring_ptr[k], ring_ptr[k + 1]) <- bucket owners[k]'s list
// (2 id + kind, bucket CSR list_ptr); one warp per request
__global__ void batcher_gather_lists_kernel(int n, const int *__restrict__ owners, const int64_t *__restrict__ list_ptr,
                                            const int *__restrict__ lists, const int *__restrict__ ring_ptr,
                                            int *__restrict__ ids, signed char *__restrict__ kinds)
{
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int64_t s0 = list_ptr[owners[w]];
    const int p0 = ring_ptr[w], cnt = ring_ptr[w + 1] - p0;
    for (int i = lane; i < cnt; i += 32) {
        const int v = lists[s0 + i];
        ids[p0 + i] = v >> 1;
        kinds[p0 + i] = (signed char)(v & 1);
    }
}

// per-batch member bounds (relative) and position -> member map from the
// ring's global CSR offsets of requests [r0, r0 + m]
__global__ void batcher_bounds_kernel(const int *__restrict__ ptr, long long r0, int m, int *__restrict__ bounds)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= m) bounds[i] = ptr[r0 + i] - ptr[r0];
}
__global__ void batcher_member_of_kernel(const int *__restrict__ bounds, int m, int *__restrict__ member_of)
{
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= m) return;
    for (int p = bounds[w] + lane; p < bounds[w + 1]; p += 32) member_of[p] = w;
}

}  // namespace gc

using namespace gc;

struct gc_batcher {
    gc_ctx *ctx = nullptr;
    gc_bh *bh = nullptr;
    gc_dm *dm = nullptr;
    TrigState st{};
    double g = 1.0, eps = 1e-4;
    // every request submitted since creation (the device ring; FIFO order)
    std::vector<int> ptr{0};  // CSR offsets of the buffer ids (host mirror of d_ptr)
    std::vector<int> owner;
    int64_t npos = 0;  // positions in the ring (ids / kinds live on the device only)
    long long head = 0;  // first pending request
    int64_t max_id = -1;
    DBuf<int> d_ids, d_ptr, d_owner, d_bounds, d_member_of;
    DBuf<signed char> d_kinds;
    // ScheduleLog rows: host part + device part ([transferred, transactions] per batch)
    struct Row {
        long long combined_id, first, count, positions;
        double emit;
        int sync_plan;
    };
    std::vector<Row> rows;
    DBuf<long long> d_rows;
    std::vector<cudaEvent_t> ev;  // 2 per batch
    long long next_combined = 0;
    int64_t fallback_plans = 0;
    // pinned staging of the submitted ids / kinds (asynchronous H2D)
    int *h_ids_pin = nullptr;
    signed char *h_kinds_pin = nullptr;
    size_t pin_cap = 0;
    ~gc_batcher()
    {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (h_ids_pin) cudaFreeHost(h_ids_pin);
        if (h_kinds_pin) cudaFreeHost(h_kinds_pin);
    }
};

namespace {

void ensure_rows(gc_batcher *b, size_t nrows)
{
    if (b->d_rows.n < 2 * nrows) {  // device rows accumulate (dm_batch_row): zero the new ones
        const size_t old = b->d_rows.n;
        b->d_rows.grow(std::max<size_t>({2 * nrows, 2 * old, 128}), b->ctx->stream);
        GC_CUDA(cudaMemsetAsync(b->d_rows.p + old, 0, (b->d_rows.n - old) * sizeof(long long), b->ctx->stream));
    }
    while (b->ev.size() < 2 * nrows) {
        cudaEvent_t e;
        GC_CUDA(cudaEventCreate(&e));
        b->ev.push_back(e);
    }
}

// size every per-batch buffer for the largest batch requests [r0, R) can form
// (windows of max_size requests over the CSR offsets ptr) before anything is
// launched: plans then never allocate (an allocation serialises host and device)
void reserve_for(gc_batcher *b, int64_t r0, int64_t R, const int *ptr)
{
    int64_t pmax = 0;
    const int64_t ms = std::max<int64_t>(1, std::min<int64_t>(b->st.max_size, R - r0));
    for (int64_t r = std::max<int64_t>(0, r0); r < R; ++r)
        pmax = std::max<int64_t>(pmax, (int64_t)ptr[std::min<int64_t>(r + ms, R)] - ptr[r]);
    dm_reserve(b->dm, pmax, ms);
    b->d_bounds.resize(std::max<int64_t>(ms + 1, (int64_t)b->d_bounds.n));
    b->d_member_of.resize(std::max<int64_t>(std::max<int64_t>(pmax, 1), (int64_t)b->d_member_of.n));
    ensure_rows(b, b->rows.size() + (size_t)((R - r0 + ms - 1) / ms) + 2);
}

// one combined launch of requests [r0, r0 + k): plan, stage, member kernel
void launch_batch(gc_batcher *b, long long r0, long long k, double now)
{
    cudaStream_t s = b->ctx->stream;
    const int m = (int)k;
    const int p0 = b->ptr[r0], P = b->ptr[r0 + k] - p0;
    const size_t row = b->rows.size();
    ensure_rows(b, row + 1);
    GC_CUDA(cudaEventRecord(b->ev[2 * row], s));
    b->d_bounds.resize(m + 1);
    b->d_member_of.resize(std::max(P, 1));
    batcher_bounds_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(b->d_ptr.p, r0, m, b->d_bounds.p);
    batcher_member_of_kernel<<<grid_for(m, 8), 256, 0, s>>>(b->d_bounds.p, m, b->d_member_of.p);
    check_launch("batcher bounds");
    int sync_plan = 0;
    if (!dm_plan_async(b->dm, b->d_ids.p + p0, b->d_kinds.p + p0, P, b->d_bounds.p, b->d_member_of.p, m, b->max_id, now,
                       b->d_rows.p + 2 * row)) {
        // the plan may evict: the synchronous data-manager path (host arrays)
        sync_plan = 1;
        ++b->fallback_plans;
        std::vector<int> hid32(P);
        std::vector<signed char> kd(P);
        if (P) {
            GC_CUDA(cudaMemcpyAsync(hid32.data(), b->d_ids.p + p0, P * sizeof(int), cudaMemcpyDeviceToHost, s));
            GC_CUDA(cudaMemcpyAsync(kd.data(), b->d_kinds.p + p0, P, cudaMemcpyDeviceToHost, s));
            GC_CUDA(cudaStreamSynchronize(s));
        }
        std::vector<int64_t> hid(hid32.begin(), hid32.end()), hb(m + 1);
        for (int i = 0; i <= m; ++i) hb[i] = b->ptr[r0 + i] - p0;
        int64_t nt = 0, np = 0;
        gc_status st = gc_dm_build_plan(b->dm, hid.data(), hb.data(), m, now, &nt, &np);
        GC_REQUIRE(st == GC_OK, st, gc_last_error());
        // kinds in plan order (REUSE_SORTED sorts each member's ids, memory.py:342-347)
        std::vector<int64_t> tx(m);
        st = gc_dm_plan_get(b->dm, nullptr, nullptr, tx.data(), nullptr);
        GC_REQUIRE(st == GC_OK, st, gc_last_error());
        if (b->dm->mode == 2) {
            std::vector<std::pair<int, signed char>> pk;
            for (int i = 0; i < m; ++i) {
                pk.clear();
                for (int p = hb[i]; p < hb[i + 1]; ++p) pk.emplace_back((int)hid[p], kd[p]);
                std::stable_sort(pk.begin(), pk.end(), [](const auto &x, const auto &y) { return x.first < y.first; });
                for (int p = hb[i]; p < hb[i + 1]; ++p) kd[p] = pk[p - hb[i]].second;
            }
        }
        std::vector<int64_t> mb(b->owner.begin() + r0, b->owner.begin() + r0 + k);
        st = gc_dm_stage_bh(b->dm, b->bh);
        GC_REQUIRE(st == GC_OK, st, gc_last_error());
        st = gc_bh_run_members(b->bh, b->dm, mb.data(), m, reinterpret_cast<const int8_t *>(kd.data()), P, b->g, b->eps);
        GC_REQUIRE(st == GC_OK, st, gc_last_error());
        st = gc_dm_release(b->dm, hid.data(), P);
        GC_REQUIRE(st == GC_OK, st, gc_last_error());
        long long h[2] = {nt, 0};
        for (int64_t t : tx) h[1] += t;
        GC_CUDA(cudaMemcpy(b->d_rows.p + 2 * row, h, sizeof(h), cudaMemcpyHostToDevice));
    } else {
        dm_members_async(b->dm, b->bh, b->d_owner.p + r0, m, b->d_bounds.p, P, b->g, b->eps);
    }
    GC_CUDA(cudaEventRecord(b->ev[2 * row + 1], s));
    b->rows.push_back({b->next_combined++, r0, k, P, now, sync_plan});
}

// poll after an arrival (or a tick) at `now`: every emitted batch is launched
void poll(gc_batcher *b, double now)
{
    for (long long k; (k = trig_poll(b->st, now)) > 0;) {
        launch_batch(b, b->head, k, now);
        b->head += k;
    }
}

}  // namespace

extern "C" {

gc_status gc_batcher_create(gc_ctx *ctx, gc_bh *bh, gc_dm *dm, int64_t max_size, double timeout_factor,
                            int32_t window, double g, double eps, gc_batcher **out)
{
    return guard([&] {
        GC_REQUIRE(ctx && bh && dm && out, GC_E_VALUE, "null argument");
        GC_REQUIRE(max_size >= 1, GC_E_VALUE, "max_size must be >= 1");
        GC_REQUIRE(window >= 0 && window <= TRIG_WMAX, GC_E_VALUE, "window must be in [0, 256]");
        GC_REQUIRE(bh->have_tree, GC_E_STATE, "no particles set");
        gc_batcher *b = new gc_batcher();
        b->ctx = ctx;
        b->bh = bh;
        b->dm = dm;
        b->st.max_size = max_size;
        b->st.factor = timeout_factor;
        b->st.window = window;
        b->g = g;
        b->eps = eps;
        *out = b;
    });
}

gc_status gc_batcher_destroy(gc_batcher *b)
{
    return guard([&] { delete b; });
}

gc_status gc_batcher_submit(gc_batcher *b, int64_t n, const int64_t *owner, const double *arrival,
                            const int64_t *ptr, const int64_t *ids, const int8_t *kinds)
{
    return guard([&] {
        GC_REQUIRE(b && (n == 0 || (owner && arrival && ptr)), GC_E_VALUE, "null argument");
        if (n == 0) return;
        const auto t_in = std::chrono::steady_clock::now();
        const int64_t npos = ptr[n] - ptr[0];
        GC_REQUIRE(npos >= 0 && (npos == 0 || (ids && kinds)), GC_E_VALUE, "bad CSR");
        GC_REQUIRE(b->npos + npos < INT_MAX, GC_E_VALUE, "ring exceeds 2^31 positions");
        const int64_t r0 = (int64_t)b->owner.size(), p0 = b->npos;
        // validate + append (vectorised: one pass per array)
        const int64_t nb = b->bh->n_buckets, nn = b->bh->n_nodes;
        b->owner.resize(r0 + n);
        b->ptr.resize(r0 + n + 1);
        for (int64_t i = 0; i < n; ++i) {
            GC_REQUIRE(owner[i] >= 0 && owner[i] < nb, GC_E_VALUE, "owner is not a bucket of the tree");
            GC_REQUIRE(ptr[i + 1] >= ptr[i], GC_E_VALUE, "bad CSR");
            b->owner[r0 + i] = (int)owner[i];
            b->ptr[r0 + i + 1] = (int)(p0 + ptr[i + 1] - ptr[0]);
        }
        // ids (int64 -> int32) and kinds go straight into the pinned staging
        // (pre-faulted; the ring's only host copy is on the device)
        cudaStream_t s0 = b->ctx->stream;
        const size_t need = (size_t)npos + 2 * (size_t)n + 1;  // ids | owners | offsets
        if (b->pin_cap < need) {
            GC_CUDA(cudaStreamSynchronize(s0));  // the previous staging may still be in flight
            if (b->h_ids_pin) cudaFreeHost(b->h_ids_pin);
            if (b->h_kinds_pin) cudaFreeHost(b->h_kinds_pin);
            b->pin_cap = need;
            GC_CUDA(cudaHostAlloc((void **)&b->h_ids_pin, b->pin_cap * sizeof(int), cudaHostAllocDefault));
            GC_CUDA(cudaHostAlloc((void **)&b->h_kinds_pin, b->pin_cap, cudaHostAllocDefault));
        } else {
            GC_CUDA(cudaStreamSynchronize(s0));  // staging reuse: the last submission's copies are done
        }
        const int64_t *src = ids + ptr[0];
        int *dst = b->h_ids_pin;
        int64_t lo = INT64_MAX, hi = -1;
        for (int64_t p = 0; p < npos; ++p) {
            const int64_t id = src[p];
            lo = std::min(lo, id);
            hi = std::max(hi, id);
            dst[p] = (int)id;
        }
        GC_REQUIRE(npos == 0 || (lo >= 0 && hi < nn), GC_E_VALUE, "buffer id is not a node of the tree");
        std::memcpy(b->h_kinds_pin, kinds + ptr[0], npos);
        b->max_id = std::max<int64_t>(b->max_id, hi);
        b->npos += npos;
        const auto t_app = std::chrono::steady_clock::now();
        cudaStream_t s = b->ctx->stream;
        // the new requests join the device ring (ids, kinds, owners, offsets);
        // the bulk (ids, kinds) goes through pinned staging: a truly
        // asynchronous copy (a pageable one blocks the host)
        b->d_ids.grow(b->npos, s);
        b->d_kinds.grow(b->npos, s);
        b->d_owner.grow(b->owner.size(), s);
        b->d_ptr.grow(b->ptr.size(), s);
        GC_CUDA(cudaMemcpyAsync(b->d_ids.p + p0, b->h_ids_pin, npos * sizeof(int), cudaMemcpyHostToDevice, s));
        GC_CUDA(cudaMemcpyAsync(b->d_kinds.p + p0, b->h_kinds_pin, npos, cudaMemcpyHostToDevice, s));
        int *po = b->h_ids_pin + npos, *pp = po + n;
        std::memcpy(po, b->owner.data() + r0, n * sizeof(int));
        std::memcpy(pp, b->ptr.data() + r0, (n + 1) * sizeof(int));
        GC_CUDA(cudaMemcpyAsync(b->d_owner.p + r0, po, n * sizeof(int), cudaMemcpyHostToDevice, s));
        GC_CUDA(cudaMemcpyAsync(b->d_ptr.p + r0, pp, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
        const auto t_h2d = std::chrono::steady_clock::now();
        dm_grow_universe(b->dm, b->max_id);
        reserve_for(b, b->head, (int64_t)b->owner.size(), b->ptr.data());
        const auto tq = std::chrono::steady_clock::now();
        // Runtime.submit_work_request (hr/runtime.py:151-163) + a poll at every arrival
        for (int64_t i = 0; i < n; ++i) {
            b->st.npending += 1;
            GC_REQUIRE(!trig_observe(b->st, arrival[i]), GC_E_CLOCK, "arrival precedes the last arrival");
            poll(b, arrival[i]);
        }
        if (getenv("GC_BATCHER_PROF")) {
            const auto te = std::chrono::steady_clock::now();
            fprintf(stderr, "gc_batcher_submit: append %.3f ms, h2d %.3f ms, reserve %.3f ms, trigger + launches %.3f ms\n",
                    std::chrono::duration<double, std::milli>(t_app - t_in).count(),
                    std::chrono::duration<double, std::milli>(t_h2d - t_app).count(),
                    std::chrono::duration<double, std::milli>(tq - t_h2d).count(),
                    std::chrono::duration<double, std::milli>(te - tq).count());
        }
    });
}

// Submission without any buffer-id traffic: every request's buffers are its
// owner bucket's interaction list as the device walk left it on the device
// (gc_bh_get_lists); only owners and arrival times cross from the host.
gc_status gc_batcher_submit_walk(gc_batcher *b, int64_t n, const int64_t *owner, const double *arrival)
{
    return guard([&] {
        GC_REQUIRE(b && (n == 0 || (owner && arrival)), GC_E_VALUE, "null argument");
        if (n == 0) return;
        gc_bh *bh = b->bh;
        GC_REQUIRE(bh->dev_lists_valid && (int64_t)bh->h_list_ptr.size() == bh->n_buckets + 1, GC_E_STATE,
                   "no device-resident lists of the current walk (gc_bh_get_lists with ids)");
        const auto t_in = std::chrono::steady_clock::now();
        const int64_t r0 = (int64_t)b->owner.size(), p0 = b->npos;
        const int64_t nb = bh->n_buckets;
        b->owner.resize(r0 + n);
        b->ptr.resize(r0 + n + 1);
        int64_t pos = p0;
        for (int64_t i = 0; i < n; ++i) {
            GC_REQUIRE(owner[i] >= 0 && owner[i] < nb, GC_E_VALUE, "owner is not a bucket of the tree");
            b->owner[r0 + i] = (int)owner[i];
            pos += bh->h_list_ptr[owner[i] + 1] - bh->h_list_ptr[owner[i]];
            GC_REQUIRE(pos < INT_MAX, GC_E_VALUE, "ring exceeds 2^31 positions");
            b->ptr[r0 + i + 1] = (int)pos;
        }
        const int64_t npos = pos - p0;
        b->npos = pos;
        b->max_id = std::max<int64_t>(b->max_id, bh->n_nodes - 1);
        cudaStream_t s = b->ctx->stream;
        const size_t need = 2 * (size_t)n + 1;
        GC_CUDA(cudaStreamSynchronize(s));  // the staging of the previous submission is free
        if (b->pin_cap < need) {
            if (b->h_ids_pin) cudaFreeHost(b->h_ids_pin);
            if (b->h_kinds_pin) cudaFreeHost(b->h_kinds_pin);
            b->pin_cap = need;
            GC_CUDA(cudaHostAlloc((void **)&b->h_ids_pin, b->pin_cap * sizeof(int), cudaHostAllocDefault));
            GC_CUDA(cudaHostAlloc((void **)&b->h_kinds_pin, b->pin_cap, cudaHostAllocDefault));
        }
        b->d_ids.grow(b->npos, s);
        b->d_kinds.grow(b->npos, s);
        b->d_owner.grow(b->owner.size(), s);
        b->d_ptr.grow(b->ptr.size(), s);
        int *po = b->h_ids_pin, *pp = po + n;
        std::memcpy(po, b->owner.data() + r0, n * sizeof(int));
        std::memcpy(pp, b->ptr.data() + r0, (n + 1) * sizeof(int));
        GC_CUDA(cudaMemcpyAsync(b->d_owner.p + r0, po, n * sizeof(int), cudaMemcpyHostToDevice, s));
        GC_CUDA(cudaMemcpyAsync(b->d_ptr.p + r0, pp, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
        if (npos > 0)
            batcher_gather_lists_kernel<<<grid_for(n, 8), 256, 0, s>>>((int)n, b->d_owner.p + r0, bh->d_bptr.p,
                                                                        bh->d_list_val2.p, b->d_ptr.p + r0, b->d_ids.p,
                                                                        b->d_kinds.p);
        check_launch("batcher_gather_lists_kernel");
        const auto t_h2d = std::chrono::steady_clock::now();
        dm_grow_universe(b->dm, b->max_id);
        reserve_for(b, b->head, (int64_t)b->owner.size(), b->ptr.data());
        const auto tq = std::chrono::steady_clock::now();
        for (int64_t i = 0; i < n; ++i) {
            b->st.npending += 1;
            GC_REQUIRE(!trig_observe(b->st, arrival[i]), GC_E_CLOCK, "arrival precedes the last arrival");
            poll(b, arrival[i]);
        }
        if (getenv("GC_BATCHER_PROF")) {
            const auto te = std::chrono::steady_clock::now();
            fprintf(stderr, "gc_batcher_submit_walk: append %.3f ms, reserve %.3f ms, trigger + launches %.3f ms\n",
                    std::chrono::duration<double, std::milli>(t_h2d - t_in).count(),
                    std::chrono::duration<double, std::milli>(tq - t_h2d).count(),
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq).count());
        }
    });
}

gc_status gc_batcher_prepare(gc_batcher *b, int64_t n, const int64_t *ptr, int64_t max_id)
{
    return guard([&] {
        GC_REQUIRE(b && ptr && n >= 0, GC_E_VALUE, "null argument");
        std::vector<int> p(n + 1);
        for (int64_t i = 0; i <= n; ++i) p[i] = (int)(ptr[i] - ptr[0]);
        const int64_t npos = p[n];
        cudaStream_t s = b->ctx->stream;
        b->d_ids.grow(b->npos + npos, s);
        b->d_ids.n = b->npos;
        b->d_kinds.grow(b->npos + npos, s);
        b->d_kinds.n = b->npos;
        b->d_owner.grow(b->owner.size() + n, s);
        b->d_owner.n = b->owner.size();
        b->d_ptr.grow(b->ptr.size() + n, s);
        b->d_ptr.n = b->ptr.size();
        if (b->pin_cap < (size_t)npos + 2 * (size_t)n + 1) {
            if (b->h_ids_pin) cudaFreeHost(b->h_ids_pin);
            if (b->h_kinds_pin) cudaFreeHost(b->h_kinds_pin);
            b->pin_cap = (size_t)npos + 2 * (size_t)n + 1;
            GC_CUDA(cudaHostAlloc((void **)&b->h_ids_pin, b->pin_cap * sizeof(int), cudaHostAllocDefault));
            GC_CUDA(cudaHostAlloc((void **)&b->h_kinds_pin, b->pin_cap, cudaHostAllocDefault));
        }
        dm_grow_universe(b->dm, max_id);
        reserve_for(b, 0, n, p.data());
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_batcher_poll(gc_batcher *b, double now)
{
    return guard([&] {
        GC_REQUIRE(b, GC_E_VALUE, "null argument");
        poll(b, now);
    });
}

gc_status gc_batcher_flush(gc_batcher *b, double now)
{
    return guard([&] {
        GC_REQUIRE(b, GC_E_VALUE, "null argument");
        // end of the phase: drain in max_size chunks (hr/timeline.py:276-283)
        while (b->st.npending > 0) {
            const long long k = std::min(b->st.npending, b->st.max_size);
            b->st.npending -= k;
            launch_batch(b, b->head, k, now);
            b->head += k;
        }
    });
}

gc_status gc_batcher_sync(gc_batcher *b, int64_t *n_batches)
{
    return guard([&] {
        GC_REQUIRE(b, GC_E_VALUE, "null argument");
        GC_CUDA(cudaStreamSynchronize(b->ctx->stream));
        const int err = dm_async_errors(b->dm);
        GC_REQUIRE(!(err & 1), GC_E_CAPACITY, "device heap full (asynchronous plan)");
        GC_REQUIRE(!(err & ~1), GC_E_VALUE, "bucket larger than a slot (raise slot_bytes)");
        if (n_batches) *n_batches = (int64_t)b->rows.size();
    });
}

gc_status gc_batcher_log(gc_batcher *b, int64_t *rows, double *times)
{
    return guard([&] {
        GC_REQUIRE(b, GC_E_VALUE, "null argument");
        GC_CUDA(cudaStreamSynchronize(b->ctx->stream));
        const size_t nb = b->rows.size();
        std::vector<long long> dr(2 * nb);
        if (nb) b->d_rows.download(dr.data(), 2 * nb, b->ctx->stream);
        GC_CUDA(cudaStreamSynchronize(b->ctx->stream));
        for (size_t i = 0; i < nb; ++i) {
            const auto &r = b->rows[i];
            if (rows) {
                int64_t *o = rows + 7 * i;
                o[0] = r.combined_id;
                o[1] = r.first;
                o[2] = r.count;
                o[3] = r.positions;
                o[4] = dr[2 * i];  // buffers transferred
                o[5] = dr[2 * i + 1];  // transactions
                o[6] = r.sync_plan;
            }
            if (times) {
                float ms = 0.f;
                GC_CUDA(cudaEventElapsedTime(&ms, b->ev[2 * i], b->ev[2 * i + 1]));
                times[2 * i] = r.emit;
                times[2 * i + 1] = ms;
            }
        }
    });
}

gc_status gc_batcher_trigger_device(int64_t max_size, double timeout_factor, int32_t window, int64_t n,
                                    const double *arrival, const int8_t *is_poll, int64_t *e_first, int64_t *e_count, double *e_time,
                                    int64_t *n_emit)
{
    return guard([&] {
        GC_REQUIRE(max_size >= 1 && window >= 0 && window <= TRIG_WMAX && n >= 0 && n_emit, GC_E_VALUE, "bad argument");
        TrigState st{};
        st.max_size = max_size;
        st.factor = timeout_factor;
        st.window = window;
        DBuf<TrigState> d_st;
        d_st.upload(&st, 1, 0);
        DBuf<double> d_t;
        if (arrival && n) d_t.upload(arrival, n, 0);
        DBuf<signed char> d_p;
        if (is_poll && n) d_p.upload(reinterpret_cast<const signed char *>(is_poll), n, 0);
        const size_t cap = std::max<int64_t>(n, 1);
        DBuf<long long> d_f, d_c;
        DBuf<double> d_e;
        DBuf<int> d_n;
        d_f.resize(cap);
        d_c.resize(cap);
        d_e.resize(cap);
        d_n.resize(2);
        d_n.zero(0);
        batcher_trigger_kernel<<<1, 1>>>(d_st.p, 0, (int)n, arrival ? d_t.p : nullptr, is_poll ? d_p.p : nullptr, d_f.p, d_c.p, d_e.p, d_n.p,
                                         d_n.p + 1);
        check_launch("batcher_trigger_kernel");
        int hn[2];
        d_n.download(hn, 2, 0);
        GC_CUDA(cudaDeviceSynchronize());
        GC_REQUIRE(!hn[1], GC_E_CLOCK, "arrival precedes the last arrival");
        std::vector<long long> f(hn[0]), c(hn[0]);
        std::vector<double> e(hn[0]);
        if (hn[0]) {
            d_f.download(f.data(), hn[0], 0);
            d_c.download(c.data(), hn[0], 0);
            d_e.download(e.data(), hn[0], 0);
        }
        GC_CUDA(cudaDeviceSynchronize());
        for (int i = 0; i < hn[0]; ++i) {
            if (e_first) e_first[i] = f[i];
            if (e_count) e_count[i] = c[i];
            if (e_time) e_time[i] = e[i];
        }
        *n_emit = hn[0];
    });
}

}  // extern "C"
