// Test infrastructure (oracle/_ref build only): a C entry surface over the
// reference's own lkv:: functions (compiled unmodified from /root/reference),
// so tests/ can check the oracle restatement bit-for-bit against them.
// Exceptions map onto the same status codes as include/lkv_b200.h.

#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include "lkv/checkpoint.hpp"
#include "lkv/errors.hpp"
#include "lkv/policy.hpp"
#include "lkv/soft_topk.hpp"

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const lkv::contract_error&) {
        return 1;
    } catch (const lkv::numeric_error&) {
        return 2;
    } catch (const lkv::budget_error&) {
        return 3;
    } catch (const lkv::overflow_guard_error&) {
        return 4;
    } catch (const lkv::degenerate_mask_error&) {
        return 5;
    } catch (...) {
        return 99;
    }
}

}  // namespace

extern "C" {

int ref_solve_threshold(const double* x, int n, double k, double* lambda, int* m) {
    return guarded([&] {
        auto [l, mm] = lkv::solve_threshold(std::span<const double>(x, static_cast<size_t>(n)), k);
        *lambda = l;
        *m = mm;
    });
}

int ref_soft_topk_forward(const double* x, int n, double k, double tau, double* values, double* lambda,
                          int* m) {
    return guarded([&] {
        auto out = lkv::soft_topk_forward(std::span<const double>(x, static_cast<size_t>(n)), k, tau);
        std::memcpy(values, out.values.data(), sizeof(double) * out.values.size());
        *lambda = out.threshold_lambda;
        *m = out.split_m;
    });
}

int ref_allocate_budgets(const double* logits, int n_layers, int n_kv_heads, double ratio, double* ratios) {
    return guarded([&] {
        const int n = n_layers * n_kv_heads;
        lkv::Tensor s = lkv::Tensor::from({n}, std::vector<double>(logits, logits + n));
        lkv::BudgetTable t = lkv::allocate_budgets(s, ratio, n_layers, n_kv_heads);
        std::memcpy(ratios, t.ratios.data(), sizeof(double) * static_cast<size_t>(n));
    });
}

int ref_freeze_budgets(const double* ratios, int n_layers, int n_kv_heads, int t, int32_t* budgets) {
    return guarded([&] {
        const int n = n_layers * n_kv_heads;
        lkv::BudgetTable table;
        table.n_layers = n_layers;
        table.n_kv_heads = n_kv_heads;
        table.ratios = lkv::Tensor::from({n}, std::vector<double>(ratios, ratios + n));
        std::vector<int> b = lkv::freeze_budgets(table, t);
        for (int i = 0; i < n; ++i) budgets[i] = b[static_cast<size_t>(i)];
    });
}

int ref_hard_topk(const double* x, int n, int b, int32_t* mask) {
    return guarded([&] {
        std::vector<int> m = lkv::hard_topk(std::span<const double>(x, static_cast<size_t>(n)), b);
        for (int i = 0; i < n; ++i) mask[i] = m[static_cast<size_t>(i)];
    });
}

// Reference-mode scorer ([k;v] -> hidden -> 1, SiLU, no output bias).
int ref_token_scores(const double* k, const double* v, int t, int d, const double* w1, const double* b1,
                     const double* w2, int hidden, double* out) {
    return guarded([&] {
        lkv::Mlp2 m;
        m.w1 = lkv::Tensor::from({2 * d, hidden}, std::vector<double>(w1, w1 + 2 * d * hidden));
        m.b1 = lkv::Tensor::from({hidden}, std::vector<double>(b1, b1 + hidden));
        m.w2 = lkv::Tensor::from({hidden, 1}, std::vector<double>(w2, w2 + hidden));
        lkv::Tensor K = lkv::Tensor::from({t, d}, std::vector<double>(k, k + static_cast<size_t>(t) * d));
        lkv::Tensor V = lkv::Tensor::from({t, d}, std::vector<double>(v, v + static_cast<size_t>(t) * d));
        lkv::Tensor u = lkv::token_scores(K, V, m);
        std::memcpy(out, u.data(), sizeof(double) * static_cast<size_t>(t));
    });
}

// Writes a real LKV policy checkpoint with the reference's own init + save path
// (policy.cpp:88-104, checkpoint.cpp:56-66) -- the trained-policy artifact of `lkv train`.
int ref_write_lkv_params(const char* path, int n_layers, int n_kv_heads, int head_dim, int d_e, unsigned long long seed) {
    return guarded([&] {
        lkv::ModelConfig cfg;
        cfg.n_layers = n_layers;
        cfg.n_kv_heads = n_kv_heads;
        cfg.n_query_heads = n_kv_heads;
        cfg.head_dim = head_dim;
        lkv::LkvParams p = lkv::init_lkv_params(cfg, seed, d_e);
        lkv::save_lkv_params(path, p);
    });
}

// load_lkv_params + head_scores (policy.cpp:106-108): the LKV-H logits of a checkpoint.
int ref_head_scores(const char* path, double* out, int n) {
    return guarded([&] {
        lkv::LkvParams p = lkv::load_lkv_params(path);
        lkv::Tensor s = lkv::head_scores(p);
        if ((int)s.numel() != n) throw lkv::contract_error("ref_head_scores: size");
        std::memcpy(out, s.data(), sizeof(double) * (size_t)n);
    });
}

}  // extern "C"
