// abi.cu -- context, device/kernel specs and the hr/kernels.py entry points.
//
// The hr/kernels.py functions (forces_from_points, direct_forces,
// md_cross_forces, md_self_forces, count_address_runs; hr/kernels.py:40-216)
// are exposed with their float64 semantics: one thread per output row, the
// reference's loop order and separately rounded float64 operations
// (__dmul_rn/__dadd_rn, no contraction), so results equal the numba kernels
// bit for bit.  They are the per-call API; the throughput path is bh.cu / md.cu.
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace gc {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

void bh_kernel_spec(const char *cls, int64_t out[5]);  // bh.cu
void md_kernel_spec(const char *cls, int64_t out[5]);  // md.cu
void dm_kernel_spec(const char *cls, int64_t out[5]);  // dm.cu (ewald_member)

constexpr int TPB = 128;

// _forces_from_points_loop (kernels.py:70-88)
__global__ void ffp_kernel(int64_t n, int64_t m, int dim, const double *__restrict__ pp, const double *__restrict__ pm,
                           const double *__restrict__ sp, const double *__restrict__ sm, double g, double eps,
                           double *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc[3] = {0.0, 0.0, 0.0};
    double xi[3];
    for (int k = 0; k < dim; ++k) xi[k] = pp[i * dim + k];
    const double gm = __dmul_rn(g, pm[i]);
    for (int64_t j = 0; j < m; ++j) {
        double r2 = __dmul_rn(eps, eps);
        bool same = true;
        for (int k = 0; k < dim; ++k) {
            const double dx = __dsub_rn(sp[j * dim + k], xi[k]);
            r2 = __dadd_rn(r2, __dmul_rn(dx, dx));
            same = same && (dx == 0.0);
        }
        if (same) continue;
        const double inv = __ddiv_rn(__dmul_rn(gm, sm[j]), __dmul_rn(r2, __dsqrt_rn(r2)));
        for (int k = 0; k < dim; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(__dsub_rn(sp[j * dim + k], xi[k]), inv));
    }
    for (int k = 0; k < dim; ++k) out[i * dim + k] = acc[k];
}

// _direct_forces_loop (kernels.py:40-54)
__global__ void direct_kernel(int64_t n, int dim, const double *__restrict__ p, const double *__restrict__ m, double g,
                              double eps, double *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc[3] = {0.0, 0.0, 0.0};
    double xi[3];
    for (int k = 0; k < dim; ++k) xi[k] = p[i * dim + k];
    const double gm = __dmul_rn(g, m[i]);
    for (int64_t j = 0; j < n; ++j) {
        if (j == i) continue;
        double r2 = __dmul_rn(eps, eps);
        for (int k = 0; k < dim; ++k) {
            const double dx = __dsub_rn(p[j * dim + k], xi[k]);
            r2 = __dadd_rn(r2, __dmul_rn(dx, dx));
        }
        const double inv = __ddiv_rn(__dmul_rn(gm, m[j]), __dmul_rn(r2, __dsqrt_rn(r2)));
        for (int k = 0; k < dim; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(__dsub_rn(p[j * dim + k], xi[k]), inv));
    }
    for (int k = 0; k < dim; ++k) out[i * dim + k] = acc[k];
}

__device__ __forceinline__ bool soft_pair(const double *a, const double *b, int dim, double cutoff, double c2,
                                          double stiffness, double *f)
{
    double r2 = 0.0;
    for (int k = 0; k < dim; ++k) {
        const double dx = __dsub_rn(a[k], b[k]);
        r2 = __dadd_rn(r2, __dmul_rn(dx, dx));
    }
    if (r2 >= c2 || r2 < 1e-12) return false;
    const double r = __dsqrt_rn(r2);
    const double mag = __ddiv_rn(__dmul_rn(stiffness, __dsub_rn(cutoff, r)), r);
    for (int k = 0; k < dim; ++k) f[k] = __dmul_rn(__dsub_rn(a[k], b[k]), mag);
    return true;
}

// _md_cross_forces_loop (kernels.py:105-125): rows i of fa (j order), then
// rows j of fb (i order) -- the same accumulation sequences as the loop nest.
__global__ void md_cross_kernel(int64_t na, int64_t nb, int dim, const double *__restrict__ pa,
                                const double *__restrict__ pb, double cutoff, double stiffness, double *__restrict__ fa,
                                double *__restrict__ fb)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double c2 = __dmul_rn(cutoff, cutoff);
    double f[3], acc[3] = {0.0, 0.0, 0.0};
    if (t < na) {
        for (int64_t j = 0; j < nb; ++j)
            if (soft_pair(pa + t * dim, pb + j * dim, dim, cutoff, c2, stiffness, f))
                for (int k = 0; k < dim; ++k) acc[k] = __dadd_rn(acc[k], f[k]);
        for (int k = 0; k < dim; ++k) fa[t * dim + k] = acc[k];
    } else if (t < na + nb) {
        const int64_t j = t - na;
        for (int64_t i = 0; i < na; ++i)
            if (soft_pair(pa + i * dim, pb + j * dim, dim, cutoff, c2, stiffness, f))
                for (int k = 0; k < dim; ++k) acc[k] = __dsub_rn(acc[k], f[k]);
        for (int k = 0; k < dim; ++k) fb[j * dim + k] = acc[k];
    }
}

// _md_self_forces_loop (kernels.py:138-156): row k receives -f(i,k) for i<k
// (in i order) before +f(k,j) for j>k (in j order).
__global__ void md_self_kernel(int64_t n, int dim, const double *__restrict__ p, double cutoff, double stiffness,
                               double *__restrict__ out)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double c2 = __dmul_rn(cutoff, cutoff);
    double f[3], acc[3] = {0.0, 0.0, 0.0};
    for (int64_t i = 0; i < r; ++i)
        if (soft_pair(p + i * dim, p + r * dim, dim, cutoff, c2, stiffness, f))
            for (int k = 0; k < dim; ++k) acc[k] = __dsub_rn(acc[k], f[k]);
    for (int64_t j = r + 1; j < n; ++j)
        if (soft_pair(p + r * dim, p + j * dim, dim, cutoff, c2, stiffness, f))
            for (int k = 0; k < dim; ++k) acc[k] = __dadd_rn(acc[k], f[k]);
    for (int k = 0; k < dim; ++k) out[r * dim + k] = acc[k];
}

// count_address_runs (kernels.py:168-177): a position starts a run iff it is
// the first of its group or its address is not previous+1.
__global__ void runs_kernel(int64_t n, int64_t group, const int64_t *__restrict__ a,
                            unsigned long long *__restrict__ total)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned c = 0;
    if (i < n) c = (i % group == 0 || a[i] != a[i - 1] + 1) ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, (unsigned long long)c);
}

// FFMA throughput probe: independent FMA chains (immediate-free, 3-register
// form) to measure the FP32 pipe peak the force roofline is quoted against.
__global__ void ffma_peak_kernel(int iters, float a, float b, float *out)
{
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5f) out[0] = s;
}

struct Staging {
    // pooled device scratch for the host-buffer entry points
    DBuf<double> a, b, c, d, e, f;
};

static Staging &staging(gc_ctx *ctx)
{
    static thread_local Staging s;
    (void)ctx;
    return s;
}

}  // namespace gc

using namespace gc;

extern "C" {

const char *gc_last_error(void) { return g_last_error.c_str(); }
const char *gc_version(void) { return "gcharm-b200 0.1 (sm_100a)"; }

gc_status gc_ctx_create(int device, gc_ctx **out)
{
    return guard([&] {
        GC_REQUIRE(out, GC_E_VALUE, "null argument");
        int count = 0;
        GC_CUDA(cudaGetDeviceCount(&count));
        GC_REQUIRE(device >= 0 && device < count, GC_E_VALUE, "no such CUDA device");
        GC_CUDA(cudaSetDevice(device));
        gc_ctx *c = new gc_ctx();
        c->device = device;
        GC_CUDA(cudaGetDeviceProperties(&c->prop, device));
        GC_REQUIRE(c->prop.major >= 10, GC_E_CUDA, "libgcharm is built for sm_100a (B200)");
        GC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        *out = c;
    });
}

gc_status gc_ctx_destroy(gc_ctx *ctx)
{
    return guard([&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

gc_status gc_ctx_sync(gc_ctx *ctx)
{
    return guard([&] { GC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

void *gc_ctx_stream(gc_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

gc_status gc_device_spec(gc_ctx *ctx, int64_t out[6])
{
    return guard([&] {
        const cudaDeviceProp &p = ctx->prop;
        out[0] = p.multiProcessorCount;
        out[1] = p.maxThreadsPerMultiProcessor;
        out[2] = p.maxBlocksPerMultiProcessor;
        out[3] = p.regsPerMultiprocessor;
        out[4] = (int64_t)p.sharedMemPerMultiprocessor;
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device);
        out[5] = khz;
    });
}

gc_status gc_kernel_spec(gc_ctx *ctx, const char *kernel_class, int64_t out[5])
{
    return guard([&] {
        GC_REQUIRE(ctx && kernel_class, GC_E_VALUE, "null argument");
        GC_CUDA(cudaSetDevice(ctx->device));
        if (!strcmp(kernel_class, "md") || !strcmp(kernel_class, "md_column")) md_kernel_spec(kernel_class, out);
        else if (!strcmp(kernel_class, "ewald_member") || !strcmp(kernel_class, "force_slot"))
            dm_kernel_spec(kernel_class, out);
        else bh_kernel_spec(kernel_class, out);
    });
}

gc_status gc_forces_from_points(gc_ctx *ctx, int64_t n, int64_t m, int32_t dim, const double *ppos,
                                const double *pmass, const double *spos, const double *smass, double g, double eps,
                                double *out)
{
    return guard([&] {
        GC_REQUIRE(ctx && dim >= 1 && dim <= 3, GC_E_VALUE, "bad argument");
        if (n == 0) return;
        Staging &S = staging(ctx);
        cudaStream_t s = ctx->stream;
        S.a.upload(ppos, n * dim, s);
        S.b.upload(pmass, n, s);
        S.c.upload(spos, m * dim, s);
        S.d.upload(smass, m, s);
        S.e.resize(n * dim);
        ffp_kernel<<<grid_for(n, TPB), TPB, 0, s>>>(n, m, dim, S.a.p, S.b.p, S.c.p, S.d.p, g, eps, S.e.p);
        check_launch("ffp_kernel");
        S.e.download(out, n * dim, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_direct_forces(gc_ctx *ctx, int64_t n, int32_t dim, const double *pos, const double *mass, double g,
                           double eps, double *out)
{
    return guard([&] {
        GC_REQUIRE(ctx && dim >= 1 && dim <= 3, GC_E_VALUE, "bad argument");
        if (n == 0) return;
        Staging &S = staging(ctx);
        cudaStream_t s = ctx->stream;
        S.a.upload(pos, n * dim, s);
        S.b.upload(mass, n, s);
        S.e.resize(n * dim);
        direct_kernel<<<grid_for(n, TPB), TPB, 0, s>>>(n, dim, S.a.p, S.b.p, g, eps, S.e.p);
        check_launch("direct_kernel");
        S.e.download(out, n * dim, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_md_cross_forces(gc_ctx *ctx, int64_t na, int64_t nb, int32_t dim, const double *pa, const double *pb,
                             double cutoff, double stiffness, double *fa, double *fb)
{
    return guard([&] {
        GC_REQUIRE(ctx && dim >= 1 && dim <= 3, GC_E_VALUE, "bad argument");
        if (na + nb == 0) return;
        Staging &S = staging(ctx);
        cudaStream_t s = ctx->stream;
        S.a.upload(pa, na * dim, s);
        S.b.upload(pb, nb * dim, s);
        S.e.resize(na * dim);
        S.f.resize(nb * dim);
        md_cross_kernel<<<grid_for(na + nb, TPB), TPB, 0, s>>>(na, nb, dim, S.a.p, S.b.p, cutoff, stiffness, S.e.p,
                                                                 S.f.p);
        check_launch("md_cross_kernel");
        S.e.download(fa, na * dim, s);
        S.f.download(fb, nb * dim, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_md_self_forces(gc_ctx *ctx, int64_t n, int32_t dim, const double *p, double cutoff, double stiffness,
                            double *out)
{
    return guard([&] {
        GC_REQUIRE(ctx && dim >= 1 && dim <= 3, GC_E_VALUE, "bad argument");
        if (n == 0) return;
        Staging &S = staging(ctx);
        cudaStream_t s = ctx->stream;
        S.a.upload(p, n * dim, s);
        S.e.resize(n * dim);
        md_self_kernel<<<grid_for(n, TPB), TPB, 0, s>>>(n, dim, S.a.p, cutoff, stiffness, S.e.p);
        check_launch("md_self_kernel");
        S.e.download(out, n * dim, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_measure_fp32_peak(gc_ctx *ctx, double *tflops, double *ms)
{
    return guard([&] {
        cudaStream_t s = ctx->stream;
        const int sms = ctx->prop.multiProcessorCount;
        const int blocks = sms * 8, threads = 256, iters = 4096;
        DBuf<float> o;
        o.resize(1);
        cudaEvent_t e0, e1;
        GC_CUDA(cudaEventCreate(&e0));
        GC_CUDA(cudaEventCreate(&e1));
        ffma_peak_kernel<<<blocks, threads, 0, s>>>(iters, 0.9999f, 0.0001f, o.p);  // warm-up
        GC_CUDA(cudaEventRecord(e0, s));
        ffma_peak_kernel<<<blocks, threads, 0, s>>>(iters, 0.9999f, 0.0001f, o.p);
        GC_CUDA(cudaEventRecord(e1, s));
        check_launch("ffma_peak_kernel");
        GC_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        GC_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        *tflops = flops / (t * 1e-3) / 1e12;
        *ms = t;
    });
}

gc_status gc_count_address_runs(gc_ctx *ctx, const int64_t *addresses, int64_t n, int64_t group, int64_t *out)
{
    return guard([&] {
        GC_REQUIRE(ctx && out && group >= 1, GC_E_VALUE, "bad argument");
        if (n == 0) {
            *out = 0;
            return;
        }
        cudaStream_t s = ctx->stream;
        DBuf<int64_t> a;
        a.upload(addresses, n, s);
        DBuf<unsigned long long> tot;
        tot.resize(1);
        tot.zero(s);
        runs_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, group, a.p, tot.p);
        check_launch("runs_kernel");
        unsigned long long h = 0;
        tot.download(&h, 1, s);
        GC_CUDA(cudaStreamSynchronize(s));
        *out = (int64_t)h;
    });
}

}  // extern "C"
