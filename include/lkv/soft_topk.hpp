// lkv/soft_topk.hpp -- Laplace-CDF relaxed top-k and its hard limit, declaration-compatible with
// proj/include/lkv/soft_topk.hpp:36-77.  Computed on the B200 in float64 with the reference's
// exact solve (stable descending sort, log-space prefix/suffix sums, first bracket within 1e-12):
// lkv_soft_topk_exact, lkv_f64_select and lkv_soft_topk_vjp of include/lkv_b200.h.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "lkv/tensor.hpp"

namespace lkv {

struct SoftTopKOutput {
    std::vector<double> values;         // f(x_i / tau - lambda) in (0, 1), summing to clamped_k
    double threshold_lambda = 0.0;
    int split_m = 0;                    // accepted bracket of the descending sort
    std::vector<double> density_terms;  // f'(x_i / tau - lambda) > 0
    std::vector<int> permutation;       // stable descending order of x
    double clamped_k = 0.0;
    double tau = 1.0;
};

struct GumbelNoise {
    std::vector<double> values;
    uint64_t seed = 0;
};

double laplace_cdf(double z);
std::pair<double, int> solve_threshold(std::span<const double> x, double k);
SoftTopKOutput soft_topk_forward(std::span<const double> x, double k, double tau);
std::pair<std::vector<double>, double> soft_topk_vjp(const SoftTopKOutput& saved, std::span<const double> upstream,
                                                     double tau);
// exactly b ones at the b largest scores, ties to the lowest index
std::vector<int> hard_topk(std::span<const double> x, int b);
GumbelNoise sample_gumbel(int n, uint64_t seed);

}  // namespace lkv
