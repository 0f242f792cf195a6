// Test infrastructure (oracle/_ref build only): a C entry surface over the
// reference's own lkv:: functions (compiled unmodified from /root/reference),
// so tests/ can check the oracle restatement bit-for-bit against them.
// Exceptions map onto the same status codes as include/lkv_b200.h.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include <string>

#include "lkv/attention.hpp"
#include "lkv/checkpoint.hpp"
#include "lkv/errors.hpp"
#include "lkv/evictsim.hpp"
#include "lkv/model.hpp"
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

// soft_topk_forward + soft_topk_vjp (soft_topk.cpp:111-189): values, density terms, then the
// vjp of `upstream` -> grad_x [n], grad_k
int ref_soft_topk_vjp(const double* x, int n, double k, double tau, const double* upstream, double* values,
                      double* density, double* grad_x, double* grad_k) {
    return guarded([&] {
        auto out = lkv::soft_topk_forward(std::span<const double>(x, static_cast<size_t>(n)), k, tau);
        std::memcpy(values, out.values.data(), sizeof(double) * out.values.size());
        std::memcpy(density, out.density_terms.data(), sizeof(double) * out.density_terms.size());
        auto [gx, gk] = lkv::soft_topk_vjp(out, std::span<const double>(upstream, static_cast<size_t>(n)), tau);
        std::memcpy(grad_x, gx.data(), sizeof(double) * gx.size());
        *grad_k = gk;
    });
}

// masked_attention_dense + masked_attention_vjp (attention.cpp:46-94,145-201), one head
int ref_masked_attention(const double* q, const double* k, const double* v, const double* mask, int n_q, int t,
                         int d, int causal, double scale, int pos_offset, int self_keep, const double* upstream,
                         double* out, double* dq, double* dk, double* dv, double* dmask) {
    return guarded([&] {
        lkv::AttentionCall c;
        c.n_q = n_q;
        c.t = t;
        c.d = d;
        c.queries.assign(q, q + (size_t)n_q * d);
        c.keys.assign(k, k + (size_t)t * d);
        c.values.assign(v, v + (size_t)t * d);
        if (mask) c.soft_mask.assign(mask, mask + t);
        c.causal = causal != 0;
        c.scale = scale;
        c.query_pos_offset = pos_offset;
        c.self_always_retained = self_keep != 0;
        lkv::AttentionSaved sv;
        std::vector<double> o = lkv::masked_attention_dense(c, &sv);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
        if (upstream) {
            lkv::AttentionGrads g = lkv::masked_attention_vjp(c, sv, std::vector<double>(upstream, upstream + (size_t)n_q * d));
            std::memcpy(dq, g.queries.data(), sizeof(double) * g.queries.size());
            std::memcpy(dk, g.keys.data(), sizeof(double) * g.keys.size());
            std::memcpy(dv, g.values.data(), sizeof(double) * g.values.size());
            if (mask && dmask) std::memcpy(dmask, g.soft_mask.data(), sizeof(double) * g.soft_mask.size());
        }
    });
}

// budget_table_csv (policy.cpp:301-311) of allocate_budgets(scores, ratio, L, H): the CSV text is
// copied into out (capacity cap, NUL-terminated); returns the status
int ref_budget_table_csv(const double* scores, int n_layers, int n_kv_heads, double ratio, char* out, int cap) {
    return guarded([&] {
        lkv::Tensor s = lkv::Tensor::from({n_layers * n_kv_heads}, std::vector<double>(scores, scores + n_layers * n_kv_heads));
        lkv::BudgetTable t = lkv::allocate_budgets(s, ratio, n_layers, n_kv_heads);
        const std::string csv = lkv::budget_table_csv(t);
        const size_t n = std::min<size_t>(csv.size(), (size_t)cap - 1);
        std::memcpy(out, csv.data(), n);
        out[n] = 0;
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

// ---- toy GQA model (model.cpp): init_model, named_params, forward_full, decode_step -------------
// A handle owns one lkv::ModelWeights built by the reference's init_model (model.cpp:173-198).
void* ref_model_create(int n_layers, int n_query_heads, int n_kv_heads, int head_dim, int vocab_size,
                       int max_seq_len, int mlp_hidden, unsigned long long seed) {
    lkv::ModelWeights* w = nullptr;
    guarded([&] {
        lkv::ModelConfig c;
        c.n_layers = n_layers;
        c.n_query_heads = n_query_heads;
        c.n_kv_heads = n_kv_heads;
        c.head_dim = head_dim;
        c.vocab_size = vocab_size;
        c.max_seq_len = max_seq_len;
        c.mlp_hidden = mlp_hidden;
        c.rng_seed = seed;
        w = new lkv::ModelWeights(lkv::init_model(c));
    });
    return w;
}

void ref_model_free(void* h) { delete static_cast<lkv::ModelWeights*>(h); }

static lkv::Tensor* find_param(void* h, const char* name) {
    for (auto& [n, t] : static_cast<lkv::ModelWeights*>(h)->named_params())
        if (n == name) return t;
    throw lkv::contract_error(std::string("no parameter ") + name);
}

// numel of a named parameter (model.cpp:142-163 names), or -1
long ref_model_param_numel(void* h, const char* name) {
    long n = -1;
    guarded([&] { n = (long)find_param(h, name)->numel(); });
    return n;
}

int ref_model_get(void* h, const char* name, double* out, long n) {
    return guarded([&] {
        lkv::Tensor* t = find_param(h, name);
        if ((long)t->numel() != n) throw lkv::contract_error("ref_model_get: size");
        std::memcpy(out, t->data(), sizeof(double) * (size_t)n);
    });
}

int ref_model_set(void* h, const char* name, const double* in, long n) {
    return guarded([&] {
        lkv::Tensor* t = find_param(h, name);
        if ((long)t->numel() != n) throw lkv::contract_error("ref_model_set: size");
        *t = lkv::Tensor::from(t->shape(), std::vector<double>(in, in + n));
    });
}

// forward_full (model.cpp:199-201): logits [t x vocab]; keys/values [L*H][t][d] (rotary applied)
int ref_forward_full(void* h, const int32_t* tokens, int t, double* logits, double* keys, double* values) {
    return guarded([&] {
        const lkv::ModelWeights& w = *static_cast<lkv::ModelWeights*>(h);
        lkv::ForwardTrace tr = lkv::forward_full(w, std::vector<int>(tokens, tokens + t));
        std::memcpy(logits, tr.logits.data(), sizeof(double) * tr.logits.numel());
        size_t o = 0;
        for (size_t i = 0; i < tr.keys.size(); ++i) {
            std::memcpy(keys + o, tr.keys[i].data(), sizeof(double) * tr.keys[i].numel());
            std::memcpy(values + o, tr.values[i].data(), sizeof(double) * tr.values[i].numel());
            o += tr.keys[i].numel();
        }
    });
}

// decode_step (model.cpp:209-287) run n_steps times on a cache built from arrays:
// head i (layer-major l*H+h) holds lens[i] rows at row offset row_off[i] of keys/values
// [rows][d] and positions[rows].  Outputs: logits [n_steps][vocab]; the rows each step
// appended, new_k/new_v [n_steps][L*H][d]; final tokens_seen.
int ref_decode_steps(void* h, const int32_t* lens, const int64_t* row_off, const double* keys,
                     const double* values, const int32_t* positions, int tokens_seen, const int32_t* tokens,
                     int n_steps, double* logits, double* new_k, double* new_v, int32_t* tokens_seen_out) {
    return guarded([&] {
        const lkv::ModelWeights& w = *static_cast<lkv::ModelWeights*>(h);
        const lkv::ModelConfig& c = w.config;
        const int d = c.head_dim, n = c.total_kv_heads();
        lkv::KvCache cache = lkv::make_cache(c);
        cache.tokens_seen = tokens_seen;
        for (int i = 0; i < n; ++i) {
            lkv::HeadCache& hc = cache.heads[(size_t)i];
            const size_t r0 = (size_t)row_off[i], r = (size_t)lens[i];
            hc.keys.assign(keys + r0 * d, keys + (r0 + r) * d);
            hc.values.assign(values + r0 * d, values + (r0 + r) * d);
            hc.retained_positions.assign(positions + r0, positions + r0 + r);
        }
        for (int s = 0; s < n_steps; ++s) {
            std::vector<double> lg = lkv::decode_step(w, cache, tokens[s]);
            std::memcpy(logits + (size_t)s * c.vocab_size, lg.data(), sizeof(double) * lg.size());
            for (int i = 0; i < n; ++i) {
                const lkv::HeadCache& hc = cache.heads[(size_t)i];
                const size_t last = (size_t)hc.retained() - 1;
                std::memcpy(new_k + ((size_t)s * n + i) * d, hc.keys.data() + last * d, sizeof(double) * d);
                std::memcpy(new_v + ((size_t)s * n + i) * d, hc.values.data() + last * d, sizeof(double) * d);
            }
        }
        *tokens_seen_out = cache.tokens_seen;
    });
}

// prefill_with_eviction (evictsim.cpp:95-238) with a learned selection policy whose LkvParams come
// from init_lkv_params(config, lkv_seed) (policy.cpp:84-100), or a baseline select kind
// (0 learned, 1 random, 2 recency, 3 sink_recent, 4 attn_window).  Outputs the compacted cache:
// lens [L*H], row offsets = exclusive scan of lens, keys/values [rows][d], positions [rows]; and
// report = {scoring_ops, peak_kv_values, kv_bytes_full, kv_bytes_compressed}.
int ref_prefill_with_eviction(void* h, const int32_t* tokens, int t, const int32_t* budgets, int select_kind,
                              unsigned long long lkv_seed, unsigned long long seed, int32_t* lens, double* keys,
                              double* values, int32_t* positions, double* report) {
    return guarded([&] {
        const lkv::ModelWeights& w = *static_cast<lkv::ModelWeights*>(h);
        const lkv::ModelConfig& c = w.config;
        lkv::LkvParams params = lkv::init_lkv_params(c, lkv_seed);
        lkv::EvictionPolicy pol;
        pol.budget = lkv::BudgetKind::uniform;
        const lkv::SelectKind kinds[] = {lkv::SelectKind::learned, lkv::SelectKind::random, lkv::SelectKind::recency,
                                         lkv::SelectKind::sink_recent, lkv::SelectKind::attn_window};
        pol.select = kinds[select_kind];
        pol.params = &params;
        const int n = c.total_kv_heads(), d = c.head_dim;
        auto [cache, rep] = lkv::prefill_with_eviction(w, std::vector<int>(tokens, tokens + t),
                                                       std::vector<int>(budgets, budgets + n), pol, seed);
        size_t row = 0;
        for (int i = 0; i < n; ++i) {
            const lkv::HeadCache& hc = cache.heads[(size_t)i];
            lens[i] = hc.retained();
            std::memcpy(keys + row * d, hc.keys.data(), sizeof(double) * hc.keys.size());
            std::memcpy(values + row * d, hc.values.data(), sizeof(double) * hc.values.size());
            std::memcpy(positions + row, hc.retained_positions.data(), sizeof(int32_t) * (size_t)hc.retained());
            row += (size_t)hc.retained();
        }
        report[0] = (double)rep.scoring_ops;
        report[1] = (double)rep.peak_kv_values;
        report[2] = rep.kv_bytes_full;
        report[3] = rep.kv_bytes_compressed;
    });
}

}  // extern "C"
