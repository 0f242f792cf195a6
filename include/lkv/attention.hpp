// lkv/attention.hpp -- multiplicative soft-mask attention, declaration-compatible with
// proj/include/lkv/attention.hpp:20-61 (inference entry points).  Runs on the B200 in float64
// (lkv_f64_attention): raw softmax over the admissible keys, times the mask, renormalised.
#pragma once

#include <vector>

#include "lkv/tensor.hpp"

namespace lkv {

struct AttentionCall {
    int n_q = 0;
    int t = 0;
    int d = 0;
    std::vector<double> queries;    // n_q x d
    std::vector<double> keys;       // t x d
    std::vector<double> values;     // t x d
    std::vector<double> soft_mask;  // t, or empty for all ones
    bool causal = true;
    double scale = 0.0;
    int query_pos_offset = 0;       // row r admits keys j <= offset + r when causal
    bool self_always_retained = false;
};

struct AttentionSaved {
    std::vector<double> p_raw;   // n_q x t
    std::vector<double> p;       // n_q x t
    std::vector<double> renorm;  // n_q
};

void validate_call(const AttentionCall& call);
std::vector<double> masked_attention_dense(const AttentionCall& call, AttentionSaved* saved = nullptr);
std::vector<double> masked_attention_blocked(const AttentionCall& call, int block_size);

}  // namespace lkv
