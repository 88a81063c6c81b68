// bh_tree.cpp -- host build of the bucket tree (product side).
//
// Restates build_bucket_tree + _fill_mass + _collect_buckets
// (hr/workloads/nbody.py:78-143) so node ids, bucket order, particle order and
// the float64 mass/COM bits equal the reference's:
//   * node ids are assigned level by level (the reference's BFS queue,
//     nbody.py:91-114); children are appended in octant order q, q bit k set
//     iff pos_k >= center_k (97-99), empty octants skipped (102-103);
//   * a node splits iff count > bucket_size and half_size >= 1e-9 (94);
//   * bucket mass = numpy pairwise sum of its masses (126), COM = sequential
//     column sum of pos*m, divided by the mass (127); internal nodes add
//     children in order with separately rounded products (131-135).
// Compiled with -ffp-contract=off so no multiply-add is fused.
#include "bh_tree.h"

#include <cmath>
#include <stdexcept>

namespace gc {

// numpy pairwise summation for a strided 1-D reduction (np.sum)
static double np_pairwise(const double *a, int64_t n)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        const int64_t lim = n - (n % 8);
        for (; i < lim; i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) s += a[i];
        return s;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return np_pairwise(a, h) + np_pairwise(a + h, n - h);
}

void HostTree::build(int64_t n_, int dim_, const double *pos, const double *mass, double box_, int64_t bucket)
{
    if (n_ < 1) throw std::invalid_argument("need at least one particle");
    if (bucket < 1) throw std::invalid_argument("bucket_size must be >= 1");
    if (dim_ < 1 || dim_ > 3) throw std::invalid_argument("dim must be 1..3");
    n = n_;
    dim = dim_;
    box = box_;
    bucket_size = bucket;
    center.clear(); half.clear(); first_child.clear(); n_child.clear(); pstart.clear(); pcount.clear();
    order.resize(n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    std::vector<int64_t> scratch(n);
    std::vector<uint8_t> oct(n);

    auto add_node = [&](const double *c, double h, int64_t ps, int64_t pc) {
        for (int k = 0; k < 3; ++k) center.push_back(k < dim ? c[k] : 0.0);
        half.push_back(h);
        first_child.push_back(-1);
        n_child.push_back(0);
        pstart.push_back(ps);
        pcount.push_back(pc);
    };
    double root_c[3] = {box / 2.0, box / 2.0, box / 2.0};
    add_node(root_c, box / 2.0, 0, n);

    // level-order expansion: ids grow as children are appended, so scanning
    // ids in increasing order visits nodes in BFS order
    for (int64_t id = 0; id < (int64_t)half.size(); ++id) {
        const int64_t cnt = pcount[id];
        if (cnt <= bucket_size || half[id] < 1e-9) continue;
        const int64_t s = pstart[id];
        int64_t hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const double cx = center[3 * id], cy = center[3 * id + 1], cz = center[3 * id + 2];
        for (int64_t i = 0; i < cnt; ++i) {
            const double *p = pos + order[s + i] * dim;
            unsigned q = (p[0] >= cx) ? 1u : 0u;
            if (dim > 1 && p[1] >= cy) q |= 2u;
            if (dim > 2 && p[2] >= cz) q |= 4u;
            oct[i] = (uint8_t)q;
            hist[q]++;
        }
        int64_t base[8];
        int64_t run = 0;
        for (int q = 0; q < 8; ++q) { base[q] = run; run += hist[q]; }
        int64_t cur[8];
        for (int q = 0; q < 8; ++q) cur[q] = base[q];
        for (int64_t i = 0; i < cnt; ++i) scratch[cur[oct[i]]++] = order[s + i];
        for (int64_t i = 0; i < cnt; ++i) order[s + i] = scratch[i];
        const double ch = half[id] / 2.0;
        int nc = 0;
        const int64_t first = (int64_t)half.size();
        for (int q = 0; q < (1 << dim); ++q) {
            if (!hist[q]) continue;
            double c[3];
            for (int k = 0; k < dim; ++k) c[k] = center[3 * id + k] + (((q >> k) & 1) ? 1.0 : -1.0) * ch;
            add_node(c, ch, s + base[q], hist[q]);
            ++nc;
        }
        first_child[id] = first;
        n_child[id] = nc;
        pcount[id] = 0;
    }
    const int64_t nn = (int64_t)half.size();

    // buckets in depth-first order (children in octant order)
    buckets.clear();
    std::vector<int64_t> stack;
    stack.push_back(0);
    while (!stack.empty()) {
        int64_t id = stack.back();
        stack.pop_back();
        if (first_child[id] < 0) {
            buckets.push_back(id);
            continue;
        }
        for (int c = n_child[id] - 1; c >= 0; --c) stack.push_back(first_child[id] + c);
    }

    // mass / centre of mass, children before parents (child ids > parent ids)
    node_mass.assign(nn, 0.0);
    com.assign(3 * nn, 0.0);
    std::vector<double> mb;
    for (int64_t id = nn - 1; id >= 0; --id) {
        if (first_child[id] < 0) {
            const int64_t s = pstart[id], c = pcount[id];
            mb.resize(c);
            for (int64_t i = 0; i < c; ++i) mb[i] = mass[order[s + i]];
            const double m = np_pairwise(mb.data(), c);
            node_mass[id] = m;
            for (int k = 0; k < dim; ++k) {
                double acc = pos[order[s] * dim + k] * mb[0];
                for (int64_t i = 1; i < c; ++i) {
                    const double t = pos[order[s + i] * dim + k] * mb[i];
                    acc = acc + t;
                }
                com[3 * id + k] = acc / m;
            }
        } else {
            double m = 0.0, c3[3] = {0.0, 0.0, 0.0};
            for (int c = 0; c < n_child[id]; ++c) {
                const int64_t ch = first_child[id] + c;
                m += node_mass[ch];
                for (int k = 0; k < dim; ++k) {
                    const double t = com[3 * ch + k] * node_mass[ch];
                    c3[k] = c3[k] + t;
                }
            }
            node_mass[id] = m;
            for (int k = 0; k < dim; ++k) com[3 * id + k] = c3[k] / m;
        }
    }
}

}  // namespace gc
