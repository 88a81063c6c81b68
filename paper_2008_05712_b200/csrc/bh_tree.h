// bh_tree.h -- host mirror of the device-built bucket tree (downloaded for the
// per-bucket API and the data manager; the tree is only ever built on the GPU).
#pragma once
#include <stdint.h>

#include <vector>

namespace gc {

struct HostTree {
    int64_t n = 0;
    int dim = 3;
    double box = 1.0;
    int64_t bucket_size = 8;
    // per node (level-order id); vectors of 3 are padded with 0 for dim < 3
    std::vector<double> center;  // 3 * n_nodes
    std::vector<double> half;
    std::vector<double> node_mass;
    std::vector<double> com;  // 3 * n_nodes
    std::vector<int64_t> first_child;
    std::vector<int32_t> n_child;
    std::vector<int64_t> pstart;  // range into `order` (buckets)
    std::vector<int64_t> pcount;  // 0 for internal nodes
    std::vector<int64_t> buckets;  // depth-first
    std::vector<int64_t> order;  // particle ids; buckets' ranges laid out in DFS order

    int64_t n_nodes() const { return (int64_t)half.size(); }
};

}  // namespace gc
