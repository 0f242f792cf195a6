// lkv_api.cpp -- the declaration-compatible C++ API (include/lkv/*.hpp) over the C ABI.
//
// A caller of the reference's hot-path API (proj/include/lkv/{policy,soft_topk,model,evictsim,
// attention}.hpp) recompiles against include/lkv/ and links liblkv_b200.so: same namespace, same
// signatures, same exception types, float64 like the reference -- but every numeric operator runs
// on the B200 through the C ABI (include/lkv_b200.h).  Host code here only validates arguments
// (in the reference's order, with its exception types), moves buffers and assembles results; the
// only host arithmetic is what the reference itself does as bookkeeping (seeded initialisation,
// budget-table formulas, memory accounting, the baseline policies' index rules).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>

#if defined(__GNUC__)
#pragma GCC visibility push(default)  // the reference API is exported from the -fvisibility=hidden library
#endif
#include "../../include/lkv/attention.hpp"
#include "../../include/lkv/checkpoint.hpp"
#include "../../include/lkv/errors.hpp"
#include "../../include/lkv/evictsim.hpp"
#include "../../include/lkv/policy.hpp"
#include "../../include/lkv/rng.hpp"
#include "../../include/lkv/soft_topk.hpp"
#include "../../include/lkv/tensor.hpp"
#include "../../include/lkv_b200.h"
#include "../../include/lkv_b200_dropin.hpp"

namespace lkv {

// ============================ device plumbing (file-local) ======================================
namespace {

[[noreturn]] void raise(lkv_status s, const std::string& where) {
    const std::string msg = where + ": " + lkv_last_error();
    switch (s) {
        case LKV_ERR_CONTRACT: throw contract_error(msg);
        case LKV_ERR_NUMERIC: throw numeric_error(msg);
        case LKV_ERR_BUDGET: throw budget_error(msg);
        case LKV_ERR_OVERFLOW_GUARD: throw overflow_guard_error(msg);
        case LKV_ERR_DEGENERATE_MASK: throw degenerate_mask_error(msg);
        default: throw device_error(msg);
    }
}
void ck(lkv_status s, const char* where) {
    if (s != LKV_OK) raise(s, where);
}
void cu(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw device_error(std::string(where) + ": " + cudaGetErrorString(e));
}

lkv_stream_t stream() {
    thread_local cudaStream_t s = nullptr;
    thread_local bool checked = false;
    if (!checked) {
        ck(lkv_device_check(), "B200 required");
        checked = true;
    }
    if (!s) cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    return (lkv_stream_t)s;
}
cudaStream_t cs() { return (cudaStream_t)stream(); }

// device buffer (256-byte aligned allocation, RAII)
struct Dev {
    void* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t bytes) : n(bytes) { cu(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        return *this;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <class T>
Dev up(const T* src, size_t count) {
    Dev d(sizeof(T) * count);
    if (count) cu(cudaMemcpyAsync(d.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, cs()), "upload");
    return d;
}
template <class T>
Dev up(const std::vector<T>& v) {
    return up(v.data(), v.size());
}
Dev up(const Tensor& t) { return up(t.data(), t.numel()); }

template <class T>
std::vector<T> down(const Dev& d, size_t count, size_t offset = 0) {
    std::vector<T> v(count);
    if (count)
        cu(cudaMemcpyAsync(v.data(), d.as<T>() + offset, sizeof(T) * count, cudaMemcpyDeviceToHost, cs()), "download");
    cu(cudaStreamSynchronize(cs()), "sync");
    return v;
}

struct Ws {
    Dev buf;
    size_t bytes;
    explicit Ws(size_t b = 256) : buf(std::max<size_t>(b, 256)), bytes(std::max<size_t>(b, 256)) {
        ck(lkv_workspace_init(buf.p, bytes, stream()), "workspace");
    }
    void* ptr() const { return buf.p; }
    void status(const char* where) { ck(lkv_workspace_status(buf.p, stream()), where); }
};

void reject_grad(const Tensor& t, const char* where) {
    if (t.defined() && t.requires_grad())
        throw contract_error(std::string(where) + ": this build is inference-only (input requires a gradient)");
}

Tensor make(std::vector<int> shape, std::vector<double> v) { return Tensor::from(std::move(shape), std::move(v)); }

}  // namespace

// ============================ Tensor (tensor.hpp:35-71) =========================================
Tensor::Tensor(std::vector<int> shape, bool requires_grad) : shape_(std::move(shape)), grad_(requires_grad) {
    size_t n = 1;
    for (int s : shape_) {
        if (s < 0) throw contract_error("tensor: negative extent");
        n *= static_cast<size_t>(s);
    }
    buf_ = std::make_shared<std::vector<double>>(n, 0.0);
}
Tensor Tensor::scalar(double v, bool requires_grad) { return from({}, {v}, requires_grad); }
Tensor Tensor::full(std::vector<int> shape, double v, bool requires_grad) {
    Tensor t(std::move(shape), requires_grad);
    std::fill(t.buf_->begin(), t.buf_->end(), v);
    return t;
}
Tensor Tensor::from(std::vector<int> shape, std::vector<double> values, bool requires_grad) {
    Tensor t(std::move(shape), requires_grad);
    if (values.size() != t.numel()) throw contract_error("tensor: value count does not match the shape");
    *t.buf_ = std::move(values);
    return t;
}
size_t Tensor::numel() const { return buf_ ? buf_->size() : 0; }
double Tensor::value() const {
    if (numel() != 1) throw contract_error("tensor: value() needs exactly one element");
    return (*buf_)[0];
}
Tensor Tensor::detached_clone() const {
    Tensor t;
    t.shape_ = shape_;
    if (buf_) t.buf_ = std::make_shared<std::vector<double>>(*buf_);
    return t;
}
bool grad_enabled() { return false; }
Tensor reshape(const Tensor& x, std::vector<int> shape) {
    Tensor t(std::move(shape));
    if (t.numel() != x.numel()) throw contract_error("reshape: element count must match");
    std::copy(x.data(), x.data() + x.numel(), t.data());
    return t;
}

// ============================ soft_topk.hpp =====================================================
double laplace_cdf(double z) {  // scalar formula (soft_topk.cpp:52-56)
    if (!std::isfinite(z)) throw numeric_error("laplace_cdf: non-finite input");
    return z >= 0.0 ? 1.0 - 0.5 * std::exp(-z) : 0.5 * std::exp(z);
}

namespace {
struct ExactOut {
    std::vector<double> values, density;
    std::vector<int> perm;
    double lambda = 0.0, kc = 0.0;
    int m = 0;
};
// lkv_soft_topk_exact: the reference's solve (soft_topk.cpp:58-164) on the device, fp64
ExactOut soft_topk_exact(std::span<const double> x, double k, double tau, bool want_all) {
    const int n = static_cast<int>(x.size());
    Ws ws;
    Dev X = up(x.data(), x.size());
    Dev V(sizeof(double) * n), D(sizeof(double) * n), P(sizeof(int32_t) * n), S(64);
    double* sc = S.as<double>();
    ck(lkv_soft_topk_exact(X.as<double>(), n, k, tau, V.as<double>(), want_all ? D.as<double>() : nullptr,
                           want_all ? P.as<int32_t>() : nullptr, sc, reinterpret_cast<int32_t*>(sc + 2), sc + 1,
                           ws.ptr(), ws.bytes, stream()),
       "soft_topk_forward");
    ws.status("soft_topk_forward");
    ExactOut o;
    o.values = down<double>(V, n);
    if (want_all) {
        o.density = down<double>(D, n);
        auto p = down<int32_t>(P, n);
        o.perm.assign(p.begin(), p.end());
    }
    auto s = down<double>(S, 3);
    o.lambda = s[0];
    o.kc = s[1];
    int32_t m = 0;
    std::memcpy(&m, &s[2], sizeof m);
    o.m = m;
    return o;
}
}  // namespace

std::pair<double, int> solve_threshold(std::span<const double> x, double k) {
    if (x.size() < 2) throw contract_error("solve_threshold: need at least two scores");  // soft_topk.cpp:60
    ExactOut o = soft_topk_exact(x, k, 1.0, false);
    return {o.lambda, o.m};
}

SoftTopKOutput soft_topk_forward(std::span<const double> x, double k, double tau) {
    if (!(tau > 0.0)) throw contract_error("soft_topk_forward: tau must be positive");
    if (x.empty()) throw contract_error("soft_topk_forward: empty scores");
    ExactOut o = soft_topk_exact(x, k, tau, true);
    SoftTopKOutput out;
    out.values = std::move(o.values);
    out.density_terms = std::move(o.density);
    out.permutation = std::move(o.perm);
    out.threshold_lambda = o.lambda;
    out.split_m = o.m;
    out.clamped_k = o.kc;
    out.tau = tau;
    return out;
}

std::pair<std::vector<double>, double> soft_topk_vjp(const SoftTopKOutput& saved, std::span<const double> upstream,
                                                     double tau) {
    const size_t n = saved.values.size();
    if (upstream.size() != n) throw contract_error("soft_topk_vjp: upstream length mismatch");
    if (!(tau > 0.0)) throw contract_error("soft_topk_vjp: tau must be positive");
    if (n == 1) return {{0.0}, 1.0};  // soft_topk.cpp:172
    if (saved.density_terms.size() != n) throw contract_error("soft_topk_vjp: saved state incomplete");
    Dev D = up(saved.density_terms), U = up(upstream.data(), n), GX(sizeof(double) * n), GK(sizeof(double));
    ck(lkv_soft_topk_vjp(D.as<double>(), U.as<double>(), 1, (int32_t)n, (int64_t)n, tau, GX.as<double>(),
                         GK.as<double>(), stream()),
       "soft_topk_vjp");
    auto gx = down<double>(GX, n);
    return {std::move(gx), down<double>(GK, 1)[0]};
}

namespace {
// top-b positions of one fp64 score vector on the device (lkv_f64_select)
std::vector<int32_t> select_positions(const Dev& scores, int n, int b) {
    Ws ws;
    int64_t offs_h[2] = {0, std::max(b, 0)};
    Dev offs = up(offs_h, 2), lens(sizeof(int32_t)), pos(sizeof(int32_t) * std::max(b, 1));
    int32_t bb = b;
    Dev B = up(&bb, 1);
    lkv_ragged_desc r{1, 1, LKV_F64, 0, std::max<int64_t>(b, 1), offs.as<int64_t>(), lens.as<int32_t>(), nullptr,
                      nullptr, pos.as<int32_t>()};
    ck(lkv_f64_select(scores.as<double>(), 1, n, n, B.as<int32_t>(), &r, ws.ptr(), ws.bytes, stream()), "hard_topk");
    ws.status("hard_topk");
    return down<int32_t>(pos, (size_t)b);
}
}  // namespace

std::vector<int> hard_topk(std::span<const double> x, int b) {
    const int n = static_cast<int>(x.size());
    if (b < 0 || b > n) throw budget_error("hard_topk: b outside [0, n]");  // soft_topk.cpp:193
    std::vector<int> mask(static_cast<size_t>(n), 0);
    if (n == 0 || b == 0) return mask;
    Dev X = up(x.data(), x.size());
    for (int32_t p : select_positions(X, n, b)) mask[static_cast<size_t>(p)] = 1;
    return mask;
}

GumbelNoise sample_gumbel(int n, uint64_t seed) {  // the seeded stream itself (soft_topk.cpp:203-215)
    if (n < 1) throw contract_error("sample_gumbel: n must be positive");
    GumbelNoise g;
    g.seed = seed;
    g.values.resize(static_cast<size_t>(n));
    Rng rng(seed);
    for (double& v : g.values) {
        const double u = std::min(std::max(rng.uniform(), 1e-12), 1.0 - 1e-12);
        v = -std::log(-std::log(u));
    }
    return g;
}

// ============================ attention.hpp =====================================================
void validate_call(const AttentionCall& c) {  // attention.cpp:31-44
    if (c.n_q < 1 || c.t < 1 || c.d < 1) throw contract_error("attention: empty extents");
    if (c.queries.size() != static_cast<size_t>(c.n_q) * c.d) throw contract_error("attention: query size");
    if (c.keys.size() != static_cast<size_t>(c.t) * c.d) throw contract_error("attention: key size");
    if (c.values.size() != static_cast<size_t>(c.t) * c.d) throw contract_error("attention: value size");
    if (!c.soft_mask.empty() && c.soft_mask.size() != static_cast<size_t>(c.t))
        throw contract_error("attention: mask length must equal t");
    for (double m : c.soft_mask)
        if (!(m >= 0.0) || !std::isfinite(m)) throw contract_error("attention: mask values must be finite and >= 0");
    if (c.causal && std::min(c.t, c.query_pos_offset + 1) < 1) throw contract_error("attention: first query row admits no key");
}

std::vector<double> masked_attention_dense(const AttentionCall& c, AttentionSaved* saved) {
    validate_call(c);
    Dev Q = up(c.queries), K = up(c.keys), V = up(c.values), O(sizeof(double) * c.n_q * c.d);
    Dev M = c.soft_mask.empty() ? Dev() : up(c.soft_mask);
    const size_t pt = static_cast<size_t>(c.n_q) * c.t;
    Dev PR = saved ? Dev(sizeof(double) * pt) : Dev(), PP = saved ? Dev(sizeof(double) * pt) : Dev(),
        RN = saved ? Dev(sizeof(double) * c.n_q) : Dev();
    lkv_f64_attn_desc a{};
    a.n_q_heads = 1;
    a.group = 1;
    a.n_q = c.n_q;
    a.t = c.t;
    a.head_dim = c.d;
    a.causal = c.causal;
    a.query_pos_offset = c.query_pos_offset;
    a.self_always_retained = c.self_always_retained;
    a.scale = c.scale;
    a.q = Q.as<double>();
    a.ldq = c.d;
    a.k = K.as<double>();
    a.v = V.as<double>();
    a.ldkv = c.d;
    a.mask = M.p ? M.as<double>() : nullptr;
    a.out = O.as<double>();
    a.ldo = c.d;
    a.p_raw = PR.p ? PR.as<double>() : nullptr;
    a.p = PP.p ? PP.as<double>() : nullptr;
    a.renorm = RN.p ? RN.as<double>() : nullptr;
    Ws ws;
    ck(lkv_f64_attention(&a, ws.ptr(), ws.bytes, stream()), "masked_attention_dense");
    ws.status("masked_attention_dense");
    if (saved) {
        saved->p_raw = down<double>(PR, pt);
        saved->p = down<double>(PP, pt);
        saved->renorm = down<double>(RN, c.n_q);
    }
    return down<double>(O, static_cast<size_t>(c.n_q) * c.d);
}

std::vector<double> masked_attention_blocked(const AttentionCall& c, int block_size) {
    validate_call(c);
    if (block_size < 1) throw contract_error("attention: block_size must be >= 1");
    // the device evaluates every block size with the same per-row arithmetic (equal to the dense path)
    return masked_attention_dense(c, nullptr);
}

// ============================ model.hpp =========================================================
void ModelConfig::validate() const {  // model.cpp:124-133
    if (n_layers < 1 || n_query_heads < 1 || n_kv_heads < 1 || head_dim < 1 || vocab_size < 1 || max_seq_len < 1)
        throw contract_error("model config: extents must be >= 1");
    if (n_query_heads % n_kv_heads != 0) throw contract_error("model config: n_query_heads must divide by n_kv_heads");
    if (head_dim % 2 != 0) throw contract_error("model config: head_dim must be even for rotary pairs");
}

std::vector<std::pair<std::string, Tensor*>> ModelWeights::named_params() {
    std::vector<std::pair<std::string, Tensor*>> out{{"tok_embed", &tok_embed}};
    for (size_t l = 0; l < layers.size(); ++l) {
        const std::string p = "layers." + std::to_string(l) + ".";
        LayerWeights& w = layers[l];
        for (auto [n, t] : std::initializer_list<std::pair<const char*, Tensor*>>{
                 {"wq", &w.wq}, {"wk", &w.wk}, {"wv", &w.wv}, {"wo", &w.wo}, {"attn_norm", &w.attn_norm},
                 {"mlp_norm", &w.mlp_norm}, {"w_gate", &w.w_gate}, {"w_up", &w.w_up}, {"w_down", &w.w_down}})
            out.emplace_back(p + n, t);
    }
    out.emplace_back("final_norm", &final_norm);
    out.emplace_back("lm_head", &lm_head);
    return out;
}
std::vector<Tensor*> ModelWeights::params() {
    std::vector<Tensor*> out;
    for (auto& nt : named_params()) out.push_back(nt.second);
    return out;
}
void ModelWeights::set_requires_grad(bool v) {
    for (Tensor* t : params()) t->set_requires_grad(v);
}

KvCache make_cache(const ModelConfig& config) {
    KvCache c;
    c.config = config;
    c.heads.resize(static_cast<size_t>(config.total_kv_heads()));
    return c;
}

ModelWeights init_model(const ModelConfig& config) {  // the reference's seeded init (model.cpp:173-198)
    config.validate();
    ModelWeights w;
    w.config = config;
    Rng rng(config.rng_seed);
    const int dm = config.d_model(), dkv = config.n_kv_heads * config.head_dim, ff = config.mlp_width();
    auto mat = [&](int r, int c) {
        Tensor t({r, c});
        for (size_t i = 0; i < t.numel(); ++i) t.data()[i] = 0.02 * rng.normal();
        return t;
    };
    w.tok_embed = mat(config.vocab_size, dm);
    for (int l = 0; l < config.n_layers; ++l) {
        LayerWeights lw;
        lw.wq = mat(dm, dm);
        lw.wk = mat(dm, dkv);
        lw.wv = mat(dm, dkv);
        lw.wo = mat(dm, dm);
        lw.attn_norm = Tensor::full({dm}, 1.0);
        lw.mlp_norm = Tensor::full({dm}, 1.0);
        lw.w_gate = mat(dm, ff);
        lw.w_up = mat(dm, ff);
        lw.w_down = mat(ff, dm);
        w.layers.push_back(std::move(lw));
    }
    w.final_norm = Tensor::full({dm}, 1.0);
    w.lm_head = mat(dm, config.vocab_size);
    return w;
}

namespace {

// the model's weights resident on the device for one call
struct DevModel {
    ModelConfig cfg;
    int dm, dkv, ff, d, H, Hq, L, V;
    Dev tok, fnorm, lm;
    struct Layer {
        Dev wq, wk, wv, wo, an, mn, wg, wu, wd;
    };
    std::vector<Layer> layers;
};

void need(const Tensor& t, std::vector<int> shape, const char* what) {
    if (!t.defined() || t.shape() != shape) throw contract_error(std::string("model weights: ") + what + " has the wrong shape");
    reject_grad(t, what);
}

DevModel upload_model(const ModelWeights& w) {
    const ModelConfig& c = w.config;
    c.validate();
    DevModel m;
    m.cfg = c;
    m.d = c.head_dim;
    m.H = c.n_kv_heads;
    m.Hq = c.n_query_heads;
    m.L = c.n_layers;
    m.V = c.vocab_size;
    m.dm = c.d_model();
    m.dkv = m.H * m.d;
    m.ff = c.mlp_width();
    if (m.d > 256) throw device_error("fp64 attention supports head_dim <= 256");
    if ((int)w.layers.size() != c.n_layers) throw contract_error("model weights: one LayerWeights per layer required");
    need(w.tok_embed, {m.V, m.dm}, "tok_embed");
    need(w.final_norm, {m.dm}, "final_norm");
    need(w.lm_head, {m.dm, m.V}, "lm_head");
    m.tok = up(w.tok_embed);
    m.fnorm = up(w.final_norm);
    m.lm = up(w.lm_head);
    for (const LayerWeights& lw : w.layers) {
        need(lw.wq, {m.dm, m.dm}, "wq");
        need(lw.wk, {m.dm, m.dkv}, "wk");
        need(lw.wv, {m.dm, m.dkv}, "wv");
        need(lw.wo, {m.dm, m.dm}, "wo");
        need(lw.attn_norm, {m.dm}, "attn_norm");
        need(lw.mlp_norm, {m.dm}, "mlp_norm");
        need(lw.w_gate, {m.dm, m.ff}, "w_gate");
        need(lw.w_up, {m.dm, m.ff}, "w_up");
        need(lw.w_down, {m.ff, m.dm}, "w_down");
        m.layers.push_back({up(lw.wq), up(lw.wk), up(lw.wv), up(lw.wo), up(lw.attn_norm), up(lw.mlp_norm),
                            up(lw.w_gate), up(lw.w_up), up(lw.w_down)});
    }
    return m;
}

void gemm(int M, int N, int K, const Dev& A, const Dev& B, Dev& C, bool acc, const char* where) {
    ck(lkv_f64_gemm(M, N, K, A.as<double>(), K, B.as<double>(), N, C.as<double>(), N, acc, stream()), where);
}

// activations of one forward pass over t rows
struct Act {
    Dev x, h, q, k, v, att, g, u;
    Act(int t, const DevModel& m)
        : x(sizeof(double) * t * m.dm), h(sizeof(double) * t * m.dm), q(sizeof(double) * t * m.dm),
          k(sizeof(double) * t * m.dkv), v(sizeof(double) * t * m.dkv), att(sizeof(double) * t * m.dm),
          g(sizeof(double) * t * m.ff), u(sizeof(double) * t * m.ff) {}
};

// attention half of layer l: h = rmsnorm(x); q, k, v; RoPE at pos0 + row; masked causal attention
// with the query's own position always retained (model.cpp:79-108)
void attention_block(const DevModel& m, int l, Act& a, int t, const Dev* masks, Ws& ws) {
    const auto& lw = m.layers[(size_t)l];
    ck(lkv_f64_rmsnorm(t, m.dm, a.x.as<double>(), m.dm, lw.an.as<double>(), 1e-6, a.h.as<double>(), m.dm, stream()),
       "rmsnorm");
    gemm(t, m.dm, m.dm, a.h, lw.wq, a.q, false, "wq");
    gemm(t, m.dkv, m.dm, a.h, lw.wk, a.k, false, "wk");
    gemm(t, m.dkv, m.dm, a.h, lw.wv, a.v, false, "wv");
    ck(lkv_f64_rope(t, m.H, m.d, a.k.as<double>(), m.dkv, 0, 10000.0, stream()), "rope k");
    ck(lkv_f64_rope(t, m.Hq, m.d, a.q.as<double>(), m.dm, 0, 10000.0, stream()), "rope q");
    lkv_f64_attn_desc d{};
    d.n_q_heads = m.Hq;
    d.group = m.Hq / m.H;
    d.n_q = t;
    d.t = t;
    d.head_dim = m.d;
    d.causal = 1;
    d.query_pos_offset = 0;
    d.self_always_retained = 1;
    d.scale = 1.0 / std::sqrt(static_cast<double>(m.d));
    d.q = a.q.as<double>();
    d.ldq = m.dm;
    d.k = a.k.as<double>();
    d.v = a.v.as<double>();
    d.ldkv = m.dkv;
    d.mask = masks ? masks->as<double>() + (size_t)l * m.H * t : nullptr;
    d.mask_ld = t;
    d.out = a.att.as<double>();
    d.ldo = m.dm;
    ck(lkv_f64_attention(&d, ws.ptr(), ws.bytes, stream()), "attention");
}

// the rest of layer l: x += att Wo; x += (silu(h2 Wg) * (h2 Wu)) Wd (model.cpp:109-117)
void mlp_block(const DevModel& m, int l, Act& a, int t) {
    const auto& lw = m.layers[(size_t)l];
    gemm(t, m.dm, m.dm, a.att, lw.wo, a.x, true, "wo");
    ck(lkv_f64_rmsnorm(t, m.dm, a.x.as<double>(), m.dm, lw.mn.as<double>(), 1e-6, a.h.as<double>(), m.dm, stream()),
       "rmsnorm");
    gemm(t, m.ff, m.dm, a.h, lw.wg, a.g, false, "w_gate");
    gemm(t, m.ff, m.dm, a.h, lw.wu, a.u, false, "w_up");
    ck(lkv_f64_swiglu((int64_t)t * m.ff, a.g.as<double>(), a.u.as<double>(), a.g.as<double>(), stream()), "swiglu");
    gemm(t, m.dm, m.ff, a.g, lw.wd, a.x, true, "w_down");
}

void embed(const DevModel& m, const std::vector<int>& tokens, Act& a, Ws& ws) {
    std::vector<int32_t> tk(tokens.begin(), tokens.end());
    Dev T = up(tk);
    ck(lkv_f64_embed(T.as<int32_t>(), (int32_t)tk.size(), m.tok.as<double>(), m.dm, m.V, a.x.as<double>(), ws.ptr(),
                     ws.bytes, stream()),
       "embedding");
}

void check_tokens(const ModelConfig& c, const std::vector<int>& tokens, const char* where) {
    for (int tok : tokens)
        if (tok < 0 || tok >= c.vocab_size) throw contract_error(std::string(where) + ": token id out of vocab");
}

// one head's [t x d] slice of a [t x (H*d)] device buffer -> host Tensor
Tensor head_tensor(const std::vector<double>& all, int t, int H, int d, int h) {
    Tensor out({t, d});
    for (int r = 0; r < t; ++r)
        std::copy(all.begin() + ((size_t)r * H + h) * d, all.begin() + ((size_t)r * H + h + 1) * d, out.data() + (size_t)r * d);
    return out;
}

ForwardTrace forward_core(const ModelWeights& w, const std::vector<int>& tokens, const std::vector<Tensor>* masks) {
    const ModelConfig& cfg = w.config;
    cfg.validate();
    const int t = static_cast<int>(tokens.size());
    if (t < 1) throw contract_error("forward: empty token sequence");
    if (t > cfg.max_seq_len) throw contract_error("forward: sequence exceeds max_seq_len");
    check_tokens(cfg, tokens, "forward");
    std::vector<double> mh;
    if (masks) {
        if ((int)masks->size() != cfg.total_kv_heads())
            throw contract_error("forward_masked: one mask per kv head per layer required");
        for (const Tensor& mk : *masks) {
            if (mk.rank() != 1 || mk.dim(0) != t) throw contract_error("forward_masked: mask length must equal t");
            reject_grad(mk, "forward_masked");
            mh.insert(mh.end(), mk.data(), mk.data() + t);
        }
        for (double v : mh)
            if (!(v >= 0.0) || !std::isfinite(v)) throw contract_error("attention: mask values must be finite and >= 0");
    }
    DevModel m = upload_model(w);
    Dev M = masks ? up(mh) : Dev();
    Ws ws;
    Act a(t, m);
    embed(m, tokens, a, ws);
    ForwardTrace tr;
    tr.keys.resize((size_t)cfg.total_kv_heads());
    tr.values.resize((size_t)cfg.total_kv_heads());
    for (int l = 0; l < m.L; ++l) {
        attention_block(m, l, a, t, masks ? &M : nullptr, ws);
        auto kh = down<double>(a.k, (size_t)t * m.dkv), vh = down<double>(a.v, (size_t)t * m.dkv);
        for (int h = 0; h < m.H; ++h) {
            tr.keys[(size_t)(l * m.H + h)] = head_tensor(kh, t, m.H, m.d, h);
            tr.values[(size_t)(l * m.H + h)] = head_tensor(vh, t, m.H, m.d, h);
        }
        mlp_block(m, l, a, t);
        tr.hidden.push_back(make({t, m.dm}, down<double>(a.x, (size_t)t * m.dm)));
    }
    ck(lkv_f64_rmsnorm(t, m.dm, a.x.as<double>(), m.dm, m.fnorm.as<double>(), 1e-6, a.h.as<double>(), m.dm, stream()),
       "final norm");
    Dev lg(sizeof(double) * t * m.V);
    gemm(t, m.V, m.dm, a.h, m.lm, lg, false, "lm_head");
    tr.logits = make({t, m.V}, down<double>(lg, (size_t)t * m.V));
    ws.status("forward");
    return tr;
}

// host KvCache <-> device ragged fp64 cache (one row of slack per head for the decode append)
KvCache ragged_to_cache(const ModelConfig& cfg, const Dev& offs, const Dev& lens, const Dev& K, const Dev& V,
                        const Dev& P, int n_heads, int d) {
    KvCache c = make_cache(cfg);
    c.heads.resize((size_t)n_heads);
    auto o = down<int64_t>(offs, (size_t)n_heads + 1);
    auto ln = down<int32_t>(lens, (size_t)n_heads);
    const int64_t rows = o[(size_t)n_heads];
    auto kh = down<double>(K, (size_t)rows * d), vh = down<double>(V, (size_t)rows * d);
    auto ph = down<int32_t>(P, (size_t)rows);
    for (int h = 0; h < n_heads; ++h) {
        HeadCache& hc = c.heads[(size_t)h];
        const size_t a = (size_t)o[(size_t)h], n = (size_t)ln[(size_t)h];
        hc.keys.assign(kh.begin() + a * d, kh.begin() + (a + n) * d);
        hc.values.assign(vh.begin() + a * d, vh.begin() + (a + n) * d);
        hc.retained_positions.assign(ph.begin() + a, ph.begin() + a + n);
    }
    return c;
}

}  // namespace

ForwardTrace forward_full(const ModelWeights& weights, const std::vector<int>& tokens) {
    return forward_core(weights, tokens, nullptr);
}
ForwardTrace forward_masked(const ModelWeights& weights, const std::vector<int>& tokens,
                            const std::vector<Tensor>& soft_masks) {
    return forward_core(weights, tokens, &soft_masks);
}

std::vector<double> decode_step(const ModelWeights& w, KvCache& cache, int token) {
    const ModelConfig& cfg = w.config;
    const ModelConfig& cc = cache.config;
    if (cfg.n_layers != cc.n_layers || cfg.n_query_heads != cc.n_query_heads || cfg.n_kv_heads != cc.n_kv_heads ||
        cfg.head_dim != cc.head_dim || cfg.vocab_size != cc.vocab_size || cfg.mlp_width() != cc.mlp_width())
        throw contract_error("cache/model config mismatch");
    if ((int)cache.heads.size() != cfg.total_kv_heads()) throw contract_error("decode_step: cache head count mismatch");
    if (token < 0 || token >= cfg.vocab_size) throw contract_error("decode_step: token id out of vocab");
    if (cache.tokens_seen >= cfg.max_seq_len) throw contract_error("decode_step: sequence exceeds max_seq_len");
    DevModel m = upload_model(w);
    const int pos = cache.tokens_seen, d = m.d, G = m.Hq / m.H;
    for (const HeadCache& hc : cache.heads)
        if (hc.keys.size() != (size_t)hc.retained() * d || hc.values.size() != hc.keys.size())
            throw contract_error("decode_step: head cache rows do not match head_dim");
    Ws ws;
    Act a(1, m);
    embed(m, {token}, a, ws);
    for (int l = 0; l < m.L; ++l) {
        const auto& lw = m.layers[(size_t)l];
        ck(lkv_f64_rmsnorm(1, m.dm, a.x.as<double>(), m.dm, lw.an.as<double>(), 1e-6, a.h.as<double>(), m.dm, stream()),
           "rmsnorm");
        gemm(1, m.dm, m.dm, a.h, lw.wq, a.q, false, "wq");
        gemm(1, m.dkv, m.dm, a.h, lw.wk, a.k, false, "wk");
        gemm(1, m.dkv, m.dm, a.h, lw.wv, a.v, false, "wv");
        ck(lkv_f64_rope(1, m.H, d, a.k.as<double>(), m.dkv, pos, 10000.0, stream()), "rope k");
        ck(lkv_f64_rope(1, m.Hq, d, a.q.as<double>(), m.dm, pos, 10000.0, stream()), "rope q");
        auto kn = down<double>(a.k, (size_t)m.dkv), vn = down<double>(a.v, (size_t)m.dkv);
        for (int kh = 0; kh < m.H; ++kh) {  // append, then attend over retained + new (model.cpp:240-263)
            HeadCache& hc = cache.head(l, kh);
            hc.keys.insert(hc.keys.end(), kn.begin() + (size_t)kh * d, kn.begin() + (size_t)(kh + 1) * d);
            hc.values.insert(hc.values.end(), vn.begin() + (size_t)kh * d, vn.begin() + (size_t)(kh + 1) * d);
            hc.retained_positions.push_back(pos);
            Dev K = up(hc.keys), V = up(hc.values);
            lkv_f64_attn_desc ad{};
            ad.n_q_heads = G;
            ad.group = G;
            ad.n_q = 1;
            ad.t = hc.retained();
            ad.head_dim = d;
            ad.causal = 0;
            ad.scale = 1.0 / std::sqrt(static_cast<double>(d));
            ad.q = a.q.as<double>() + (size_t)kh * G * d;
            ad.ldq = m.dm;
            ad.k = K.as<double>();
            ad.v = V.as<double>();
            ad.ldkv = d;
            ad.out = a.att.as<double>() + (size_t)kh * G * d;
            ad.ldo = m.dm;
            ck(lkv_f64_attention(&ad, ws.ptr(), ws.bytes, stream()), "decode attention");
            cu(cudaStreamSynchronize(cs()), "sync");  // K / V are released at scope end
        }
        mlp_block(m, l, a, 1);
    }
    ck(lkv_f64_rmsnorm(1, m.dm, a.x.as<double>(), m.dm, m.fnorm.as<double>(), 1e-6, a.h.as<double>(), m.dm, stream()),
       "final norm");
    Dev lg(sizeof(double) * m.V);
    gemm(1, m.V, m.dm, a.h, m.lm, lg, false, "lm_head");
    auto logits = down<double>(lg, (size_t)m.V);
    ws.status("decode_step");
    cache.tokens_seen = pos + 1;
    return logits;
}

KvCache cache_from_trace(const ModelConfig& config, const ForwardTrace& trace,
                         const std::vector<std::vector<int>>& hard_masks) {
    if (trace.keys.size() != static_cast<size_t>(config.total_kv_heads()))
        throw contract_error("cache_from_trace: trace head count mismatch");
    if (hard_masks.size() != trace.keys.size()) throw contract_error("cache_from_trace: one mask per head required");
    const int n = config.total_kv_heads(), d = config.head_dim;
    const int t = trace.keys[0].dim(0);
    std::vector<double> kh, vh;
    std::vector<int32_t> mk;
    for (int i = 0; i < n; ++i) {
        const auto& m = hard_masks[(size_t)i];
        if (static_cast<int>(m.size()) != t) throw contract_error("cache_from_trace: mask length mismatch");
        const Tensor& k = trace.keys[(size_t)i];
        const Tensor& v = trace.values[(size_t)i];
        if (k.numel() != (size_t)t * d || v.numel() != (size_t)t * d)
            throw contract_error("cache_from_trace: trace rows do not match head_dim");
        kh.insert(kh.end(), k.data(), k.data() + k.numel());
        vh.insert(vh.end(), v.data(), v.data() + v.numel());
        mk.insert(mk.end(), m.begin(), m.end());
    }
    Dev K = up(kh), V = up(vh), MK = up(mk);
    int32_t tl = t;
    lkv_cache_desc cd{1, config.n_layers, config.n_kv_heads, d, t, LKV_F64, 0, K.p, V.p, &tl};
    Ws ws(lkv_workspace_bytes(&cd, 1));
    Dev cnt(sizeof(int32_t) * n);
    ck(lkv_mask_counts(&cd, MK.as<int32_t>(), t, cnt.as<int32_t>(), ws.ptr(), ws.bytes, stream()), "cache_from_trace");
    int64_t rows = 0;
    for (int32_t c : down<int32_t>(cnt, (size_t)n)) rows += c;
    Dev offs(sizeof(int64_t) * (n + 1)), lens(sizeof(int32_t) * n), RK(sizeof(double) * std::max<int64_t>(rows, 1) * d),
        RV(sizeof(double) * std::max<int64_t>(rows, 1) * d), RP(sizeof(int32_t) * std::max<int64_t>(rows, 1));
    lkv_ragged_desc r{n, d, LKV_F64, 0, rows, offs.as<int64_t>(), lens.as<int32_t>(), RK.p, RV.p, RP.as<int32_t>()};
    ck(lkv_cache_from_trace(&cd, MK.as<int32_t>(), t, &r, ws.ptr(), ws.bytes, stream()), "cache_from_trace");
    ws.status("cache_from_trace");
    KvCache c = ragged_to_cache(config, offs, lens, RK, RV, RP, n, d);
    c.tokens_seen = t;
    return c;
}

// ============================ policy.hpp ========================================================
namespace {
Mlp2 init_mlp2(Rng& rng, int in, int hidden) {  // policy.cpp:18-28
    Mlp2 m;
    m.w1 = Tensor({in, hidden});
    m.b1 = Tensor({hidden});
    m.w2 = Tensor({hidden, 1});
    const double g1 = 1.0 / std::sqrt(static_cast<double>(in)), g2 = 1.0 / std::sqrt(static_cast<double>(hidden));
    for (size_t i = 0; i < m.w1.numel(); ++i) m.w1.data()[i] = g1 * rng.normal();
    for (size_t i = 0; i < m.w2.numel(); ++i) m.w2.data()[i] = g2 * rng.normal();
    return m;
}

// mlp2_forward on the device (policy.cpp:30-34): x [t x (input * d)] as k (and v) parts
std::vector<double> mlp2_device(const Mlp2& m, const double* k, const double* v, int t, int d, int input) {
    reject_grad(m.w1, "token scorer");
    reject_grad(m.b1, "token scorer");
    reject_grad(m.w2, "token scorer");
    const int in = input * d;
    if (m.w1.rank() != 2 || m.w1.dim(0) != in) throw contract_error("matmul: inner dimensions differ");
    const int hidden = m.w1.dim(1);
    if (m.b1.numel() != (size_t)hidden || m.w2.numel() != (size_t)hidden)
        throw contract_error("token scorer: b1 / w2 do not match the hidden width");
    if (t == 0) return {};
    Dev K = up(k, (size_t)t * d), V = v ? up(v, (size_t)t * d) : Dev(), W1 = up(m.w1), B1 = up(m.b1), W2 = up(m.w2),
        U(sizeof(double) * t);
    Ws ws;
    ck(lkv_f64_token_scores(t, d, input, K.as<double>(), d, v ? V.as<double>() : nullptr, d, W1.as<double>(),
                            B1.as<double>(), W2.as<double>(), hidden, LKV_ACT_SILU, U.as<double>(), ws.ptr(), ws.bytes,
                            stream()),
       "token_scores");
    ws.status("token_scores");
    return down<double>(U, (size_t)t);
}

void clamp_and_renormalize(std::vector<double>& r, double target_sum) {  // policy.cpp:37-57
    const double lo = 1e-6, hi = 1.0 - 1e-6;
    for (int pass = 0; pass < 16; ++pass) {
        double fixed = 0.0, free_sum = 0.0;
        bool out = false;
        for (double v : r) {
            if (v >= hi || v <= lo) fixed += std::clamp(v, lo, hi);
            else free_sum += v;
            out |= v > hi || v < lo;
        }
        if (!out) break;
        const double f = free_sum > 0.0 ? (target_sum - fixed) / free_sum : 1.0;
        for (double& v : r) v = v > hi ? hi : (v < lo ? lo : v * f);
    }
}
}  // namespace

std::vector<std::pair<std::string, Tensor*>> LkvParams::named_params() {
    std::vector<std::pair<std::string, Tensor*>> out{{"head_embeddings", &head_embeddings},
                                                     {"head_predictor.w1", &head_predictor.w1},
                                                     {"head_predictor.b1", &head_predictor.b1},
                                                     {"head_predictor.w2", &head_predictor.w2}};
    for (size_t i = 0; i < token_scorers.size(); ++i) {
        const std::string p = "token_scorers." + std::to_string(i) + ".";
        out.emplace_back(p + "w1", &token_scorers[i].w1);
        out.emplace_back(p + "b1", &token_scorers[i].b1);
        out.emplace_back(p + "w2", &token_scorers[i].w2);
    }
    return out;
}
std::vector<Tensor*> LkvParams::params() {
    std::vector<Tensor*> out;
    for (auto& nt : named_params()) out.push_back(nt.second);
    return out;
}
void LkvParams::set_requires_grad(bool v) {
    for (Tensor* t : params()) t->set_requires_grad(v);
}

LkvParams init_lkv_params(const ModelConfig& config, uint64_t seed, int d_e) {  // policy.cpp:84-100
    config.validate();
    LkvParams p;
    p.n_layers = config.n_layers;
    p.n_kv_heads = config.n_kv_heads;
    p.d_head = config.head_dim;
    p.d_e = d_e > 0 ? d_e : config.head_dim;
    if (p.d_e % 2 != 0) throw contract_error("init_lkv_params: d_e must be even");
    Rng rng(seed);
    p.head_embeddings = Tensor({p.total_heads(), p.d_e});
    for (size_t i = 0; i < p.head_embeddings.numel(); ++i) p.head_embeddings.data()[i] = 0.1 * rng.normal();
    p.head_predictor = init_mlp2(rng, p.d_e, p.d_e / 2);
    for (int h = 0; h < p.total_heads(); ++h) p.token_scorers.push_back(init_mlp2(rng, 2 * p.d_head, p.d_head));
    return p;
}

Tensor head_scores(const LkvParams& params) {  // policy.cpp:106-108, on the device
    const Tensor& e = params.head_embeddings;
    reject_grad(e, "head_scores");
    if (e.rank() != 2) throw contract_error("head_scores: embeddings must be rank-2");
    const int n = e.dim(0);
    auto u = mlp2_device(params.head_predictor, e.data(), nullptr, n, e.dim(1), LKV_SCORER_K);
    return make({n}, std::move(u));
}

BudgetTable allocate_budgets(const Tensor& scores, double target_ratio, int n_layers, int n_kv_heads) {
    if (!(target_ratio > 0.0 && target_ratio < 1.0)) throw budget_error("target ratio must lie in (0,1)");
    const int n = n_layers * n_kv_heads;
    if (scores.rank() != 1 || scores.dim(0) != n) throw contract_error("allocate_budgets: score length mismatch");
    reject_grad(scores, "allocate_budgets");
    BudgetTable table;
    table.n_layers = n_layers;
    table.n_kv_heads = n_kv_heads;
    table.target_ratio = target_ratio;
    // soft_topk(scores, k = R n, tau = 1) (policy.cpp:118): the exact solve on the device
    ExactOut o = soft_topk_exact(std::span<const double>(scores.data(), scores.numel()), target_ratio * n, 1.0, false);
    table.ratios = make({n}, std::move(o.values));
    return table;
}

std::vector<int> freeze_budgets(const BudgetTable& table, int t) {  // floor(r t) on the device (K2 freeze)
    if (t < 1) throw contract_error("freeze_budgets: t must be >= 1");
    const int n = table.n_layers * table.n_kv_heads;
    if (!table.ratios.defined() || table.ratios.numel() != (size_t)n)
        throw contract_error("freeze_budgets: ratio table size mismatch");
    if (n == 0) return {};
    Dev R = up(table.ratios), B(sizeof(int32_t) * n);
    int32_t tl = t;
    Ws ws;
    ck(lkv_freeze_budgets(R.as<double>(), n, 0.5, LKV_BUDGET_FLOOR, &tl, 1, 0, B.as<int32_t>(), nullptr, ws.ptr(),
                          ws.bytes, stream()),
       "freeze_budgets");
    ws.status("freeze_budgets");
    auto b = down<int32_t>(B, (size_t)n);
    return std::vector<int>(b.begin(), b.end());
}

Tensor token_scores(const Tensor& keys, const Tensor& values, const Mlp2& scorer) {
    if (keys.rank() != 2 || values.rank() != 2 || keys.dim(0) != values.dim(0))
        throw contract_error("token_scores: keys/values must be rank-2 with equal first extents");
    if (keys.dim(1) != values.dim(1)) throw device_error("token_scores: keys and values of different widths");
    reject_grad(keys, "token_scores");
    reject_grad(values, "token_scores");
    const int t = keys.dim(0);
    auto u = mlp2_device(scorer, keys.data(), values.data(), t, keys.dim(1), LKV_SCORER_KV);
    return make({t}, std::move(u));
}

std::vector<int> inference_select(std::span<const double> u, int b) { return hard_topk(u, b); }

BudgetKind budget_kind_from_string(const std::string& s) {
    if (s == "learned") return BudgetKind::learned;
    if (s == "uniform") return BudgetKind::uniform;
    if (s == "pyramid") return BudgetKind::pyramid;
    if (s == "binary_heads") return BudgetKind::binary_heads;
    throw contract_error("unknown budget policy: " + s);
}
SelectKind select_kind_from_string(const std::string& s) {
    if (s == "learned") return SelectKind::learned;
    if (s == "random") return SelectKind::random;
    if (s == "recency") return SelectKind::recency;
    if (s == "sink_recent") return SelectKind::sink_recent;
    if (s == "attn_window") return SelectKind::attn_window;
    throw contract_error("unknown selection policy: " + s);
}
std::string to_string(BudgetKind k) {
    switch (k) {
        case BudgetKind::learned: return "learned";
        case BudgetKind::uniform: return "uniform";
        case BudgetKind::pyramid: return "pyramid";
        case BudgetKind::binary_heads: return "binary_heads";
    }
    return "?";
}
std::string to_string(SelectKind k) {
    switch (k) {
        case SelectKind::learned: return "learned";
        case SelectKind::random: return "random";
        case SelectKind::recency: return "recency";
        case SelectKind::sink_recent: return "sink_recent";
        case SelectKind::attn_window: return "attn_window";
    }
    return "?";
}

BudgetTable baseline_budget(BudgetKind kind, int n_layers, int n_kv_heads, double target_ratio, double high_fraction) {
    if (!(target_ratio > 0.0 && target_ratio < 1.0)) throw budget_error("target ratio must lie in (0,1)");
    const int n = n_layers * n_kv_heads;
    const double total = target_ratio * n;
    std::vector<double> r((size_t)n, target_ratio);
    if (kind == BudgetKind::pyramid) {  // weight L - l per layer, sum preserved (policy.cpp:236-243)
        const double wsum = n_layers * (n_layers + 1) / 2.0;
        for (int l = 0; l < n_layers; ++l)
            for (int h = 0; h < n_kv_heads; ++h)
                r[(size_t)(l * n_kv_heads + h)] = target_ratio * n_layers * (n_layers - l) / wsum;
    } else if (kind == BudgetKind::binary_heads) {  // high heads at 5x the low ratio (:244-250)
        const int n_high = static_cast<int>(std::ceil(high_fraction * n));
        const double low = total / (n + 4.0 * n_high);
        for (int i = 0; i < n; ++i) r[(size_t)i] = i < n_high ? 5.0 * low : low;
    } else if (kind == BudgetKind::learned) {
        throw contract_error("baseline_budget: learned budgets come from allocate_budgets");
    }
    clamp_and_renormalize(r, total);
    BudgetTable t;
    t.n_layers = n_layers;
    t.n_kv_heads = n_kv_heads;
    t.target_ratio = target_ratio;
    t.ratios = make({n}, std::move(r));
    return t;
}

std::vector<int> baseline_select(SelectKind kind, const SelectContext& ctx, int b, uint64_t rng_seed) {
    const int t = ctx.t;
    if (b < 0 || b > t) throw budget_error("baseline_select: b outside [0, t]");
    std::vector<int> mask((size_t)t, 0);
    switch (kind) {
        case SelectKind::random: {  // seeded Fisher-Yates (policy.cpp:258-266)
            std::vector<int> idx((size_t)t);
            std::iota(idx.begin(), idx.end(), 0);
            Rng rng(rng_seed);
            for (int i = t - 1; i > 0; --i) std::swap(idx[(size_t)i], idx[(size_t)rng.uniform_int(0, i + 1)]);
            for (int i = 0; i < b; ++i) mask[(size_t)idx[(size_t)i]] = 1;
            return mask;
        }
        case SelectKind::recency:
            for (int j = t - b; j < t; ++j) mask[(size_t)j] = 1;
            return mask;
        case SelectKind::sink_recent: {
            const int sinks = std::min(4, b);
            for (int j = 0; j < sinks; ++j) mask[(size_t)j] = 1;
            for (int j = t - (b - sinks); j < t; ++j) mask[(size_t)j] = 1;
            return mask;
        }
        case SelectKind::attn_window: {  // mean attention from the window rows, on the device (:276-303)
            if (!ctx.keys || ctx.d <= 0) throw contract_error("attn_window: context with keys required");
            const int rows = (int)ctx.window_positions.size();
            if (rows == 0) throw contract_error("attn_window: no window rows");
            Dev K = up(*ctx.keys), Q = up(ctx.window_queries), O(sizeof(double) * ctx.d),
                PR(sizeof(double) * (size_t)t), R(sizeof(double) * (size_t)t);
            cu(cudaMemsetAsync(R.p, 0, sizeof(double) * (size_t)t, cs()), "memset");
            Ws ws;
            std::vector<double> received((size_t)t, 0.0);
            for (int r = 0; r < rows; ++r) {
                lkv_f64_attn_desc a{};
                a.n_q_heads = 1;
                a.group = 1;
                a.n_q = 1;
                a.t = std::min(t, ctx.window_positions[(size_t)r] + 1);
                a.head_dim = ctx.d;
                a.scale = ctx.scale;
                a.q = Q.as<double>() + (size_t)r * ctx.d;
                a.ldq = ctx.d;
                a.k = K.as<double>();
                a.v = K.as<double>();
                a.ldkv = ctx.d;
                a.out = O.as<double>();
                a.ldo = ctx.d;
                a.p_raw = PR.as<double>();
                ck(lkv_f64_attention(&a, ws.ptr(), ws.bytes, stream()), "attn_window");
                auto p = down<double>(PR, (size_t)a.t);
                for (int j = 0; j < a.t; ++j) received[(size_t)j] += p[(size_t)j];
            }
            ws.status("attn_window");
            for (double& v : received) v /= rows;
            return hard_topk(received, b);
        }
        case SelectKind::learned:
            throw contract_error("baseline_select: learned selection comes from token scorers");
    }
    return mask;
}

ParamCounts param_count(int n_layers, int n_kv_heads, int d_head, int d_e) {  // policy.cpp:289-299
    if (n_layers < 1 || n_kv_heads < 1 || d_head < 1 || d_e < 1) throw contract_error("param_count: bad geometry");
    ParamCounts c;
    const int64_t heads = static_cast<int64_t>(n_layers) * n_kv_heads;
    c.embeddings = heads * d_e;
    c.head_predictor = static_cast<int64_t>(d_e) * (d_e / 2) + 2 * (d_e / 2);
    c.per_scorer = static_cast<int64_t>(2 * d_head) * d_head + 2 * d_head;
    c.scorers_total = heads * c.per_scorer;
    c.total = c.embeddings + c.head_predictor + c.scorers_total;
    return c;
}

std::string budget_table_csv(const BudgetTable& table) {  // policy.cpp:301-311
    std::string out = "layer,head,ratio\n";
    char line[64];
    for (int l = 0; l < table.n_layers; ++l)
        for (int h = 0; h < table.n_kv_heads; ++h) {
            std::snprintf(line, sizeof line, "%d,%d,%.6f\n", l, h, table.at(l, h));
            out += line;
        }
    return out;
}

// ============================ evictsim.hpp ======================================================
void MemoryModel::validate() const {
    if (n_layers < 1 || n_kv_heads < 1 || head_dim < 1 || tokens < 1 || !(bytes_per_element > 0.0))
        throw contract_error("memory model: all extents must be positive");
}

MemoryReport kv_memory_bytes(const MemoryModel& mm, double retention) {  // evictsim.cpp:56-65
    mm.validate();
    if (!(retention > 0.0) || retention > 1.0) throw budget_error("kv_memory_bytes: retention must lie in (0, 1]");
    MemoryReport r;
    r.full_bytes = static_cast<double>(mm.n_layers) * mm.n_kv_heads * mm.head_dim * 2.0 * mm.bytes_per_element *
                   static_cast<double>(mm.tokens);
    r.compressed_bytes = retention * r.full_bytes;
    r.reduction_factor = r.full_bytes / r.compressed_bytes;
    return r;
}

MemoryReport kv_memory_bytes(const MemoryModel& mm, const std::vector<int>& per_head_budgets) {  // :67-81
    mm.validate();
    if (static_cast<int>(per_head_budgets.size()) != mm.n_layers * mm.n_kv_heads)
        throw contract_error("kv_memory_bytes: one budget per head required");
    MemoryReport r;
    r.full_bytes = static_cast<double>(mm.n_layers) * mm.n_kv_heads * mm.head_dim * 2.0 * mm.bytes_per_element *
                   static_cast<double>(mm.tokens);
    double kept = 0.0;
    for (int b : per_head_budgets) kept += static_cast<double>(b);
    r.compressed_bytes = kept * mm.head_dim * 2.0 * mm.bytes_per_element;
    r.reduction_factor = r.compressed_bytes > 0.0 ? r.full_bytes / r.compressed_bytes : std::numeric_limits<double>::infinity();
    return r;
}

BudgetTable policy_budget_table(const EvictionPolicy& policy, double target_ratio, const ModelConfig& config) {
    if (policy.budget == BudgetKind::learned) {
        if (!policy.params) throw contract_error("learned budgeting needs trained parameters");
        return allocate_budgets(head_scores(*policy.params), target_ratio, config.n_layers, config.n_kv_heads);
    }
    return baseline_budget(policy.budget, config.n_layers, config.n_kv_heads, target_ratio, policy.high_fraction);
}

// Layer-by-layer prefill with eviction (evictsim.cpp:95-238) on the device: per layer the
// projections, RoPE and causal attention over the full prefix; then per KV head the scores
// (LKV-T scorer, or a baseline rule), the top-b selection and the compaction of that layer into
// the ragged cache -- only one full layer of K/V is live at a time.
std::pair<KvCache, SimReport> prefill_with_eviction(const ModelWeights& weights, const std::vector<int>& tokens,
                                                    const std::vector<int>& budgets, const EvictionPolicy& policy,
                                                    uint64_t seed) {
    const ModelConfig& cfg = weights.config;
    cfg.validate();
    const int t = static_cast<int>(tokens.size());
    if (static_cast<int>(budgets.size()) != cfg.total_kv_heads())
        throw contract_error("prefill_with_eviction: one budget per head required");
    for (int b : budgets)
        if (b < 0 || b > t) throw budget_error("prefill_with_eviction: budget outside [0, t]");
    if ((policy.select == SelectKind::learned || policy.budget == BudgetKind::learned) && !policy.params)
        throw contract_error("prefill_with_eviction: learned policy needs parameters");
    if (t < 1) throw contract_error("prefill_with_eviction: empty token sequence");
    check_tokens(cfg, tokens, "embedding_rows");
    const int H = cfg.n_kv_heads, d = cfg.head_dim;
    if (policy.select == SelectKind::learned && (int)policy.params->token_scorers.size() != cfg.total_kv_heads())
        throw contract_error("prefill_with_eviction: one token scorer per head required");

    SimReport rep;
    rep.budget_policy = to_string(policy.budget);
    rep.select_policy = to_string(policy.select);
    rep.retained_per_head.assign((size_t)cfg.total_kv_heads(), 0);
    KvCache cache = make_cache(cfg);
    cache.tokens_seen = t;
    DevModel m = upload_model(weights);
    Ws ws;
    Act a(t, m);
    embed(m, tokens, a, ws);
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    Dev Kh(sizeof(double) * (size_t)H * t * d), Vh(sizeof(double) * (size_t)H * t * d), S(sizeof(double) * (size_t)H * t);
    int32_t tl = t;
    lkv_cache_desc layer{1, 1, H, d, t, LKV_F64, 0, Kh.p, Vh.p, &tl};  // one dense layer, head-major
    Ws lws(lkv_workspace_bytes(&layer, 1));
    int64_t compressed = 0;
    double select_seconds = 0.0;
    for (int l = 0; l < m.L; ++l) {
        attention_block(m, l, a, t, nullptr, ws);
        rep.peak_kv_values = std::max(rep.peak_kv_values, compressed + static_cast<int64_t>(t) * H * d * 2);
        ck(lkv_f64_split_heads(t, H, d, a.k.as<double>(), m.dkv, Kh.as<double>(), t, stream()), "split k");
        ck(lkv_f64_split_heads(t, H, d, a.v.as<double>(), m.dkv, Vh.as<double>(), t, stream()), "split v");
        // per-layer ragged block: head kh's rows at [sum_{j<kh} b_j, ...)
        std::vector<int32_t> bl((size_t)H);
        std::vector<int64_t> offs((size_t)H + 1, 0);
        for (int kh = 0; kh < H; ++kh) {
            bl[(size_t)kh] = budgets[(size_t)(l * H + kh)];
            offs[(size_t)kh + 1] = offs[(size_t)kh] + bl[(size_t)kh];
        }
        const int64_t rows = offs[(size_t)H];
        Dev OF = up(offs), LN(sizeof(int32_t) * H), BL = up(bl), RP(sizeof(int32_t) * std::max<int64_t>(rows, 1)),
            RK(sizeof(double) * std::max<int64_t>(rows, 1) * d), RV(sizeof(double) * std::max<int64_t>(rows, 1) * d);
        lkv_ragged_desc r{H, d, LKV_F64, 0, rows, OF.as<int64_t>(), LN.as<int32_t>(), RK.p, RV.p, RP.as<int32_t>()};
        cu(cudaStreamSynchronize(cs()), "sync");
        const auto t0 = std::chrono::steady_clock::now();
        if (policy.select == SelectKind::learned) {
            for (int kh = 0; kh < H; ++kh) {  // one LKV-T scorer per (l, h) (policy.cpp:100-102)
                const Mlp2& sc = policy.params->token_scorers[(size_t)(l * H + kh)];
                reject_grad(sc.w1, "token scorer");
                if (sc.w1.rank() != 2 || sc.w1.dim(0) != 2 * d || sc.b1.numel() != (size_t)sc.w1.dim(1) ||
                    sc.w2.numel() != (size_t)sc.w1.dim(1))
                    throw contract_error("matmul: inner dimensions differ");
                const int hidden = sc.w1.dim(1);
                Dev W1 = up(sc.w1), B1 = up(sc.b1), W2 = up(sc.w2);
                ck(lkv_f64_token_scores(t, d, LKV_SCORER_KV, Kh.as<double>() + (size_t)kh * t * d, d,
                                        Vh.as<double>() + (size_t)kh * t * d, d, W1.as<double>(), B1.as<double>(),
                                        W2.as<double>(), hidden, LKV_ACT_SILU, S.as<double>() + (size_t)kh * t, ws.ptr(),
                                        ws.bytes, stream()),
                   "token_scores");
                cu(cudaStreamSynchronize(cs()), "sync");
                rep.scoring_ops += static_cast<int64_t>(t) * (2 * d * d + 3 * d);
            }
            ck(lkv_f64_select(S.as<double>(), H, t, t, BL.as<int32_t>(), &r, ws.ptr(), ws.bytes, stream()),
               "inference_select");
            ck(lkv_compact(&layer, &r, ws.ptr(), ws.bytes, stream()), "compaction");
        } else {
            std::vector<int32_t> masks;
            auto kh_all = policy.select == SelectKind::attn_window ? down<double>(Kh, (size_t)H * t * d) : std::vector<double>();
            auto q_all = policy.select == SelectKind::attn_window ? down<double>(a.q, (size_t)t * m.dm) : std::vector<double>();
            for (int kh = 0; kh < H; ++kh) {
                SelectContext ctx;
                ctx.t = t;
                ctx.d = d;
                std::vector<double> keys_raw;
                if (policy.select == SelectKind::attn_window) {
                    keys_raw.assign(kh_all.begin() + (size_t)kh * t * d, kh_all.begin() + (size_t)(kh + 1) * t * d);
                    const int w = std::min(policy.window, t), G = cfg.group_size();
                    for (int qh = kh * G; qh < (kh + 1) * G; ++qh)
                        for (int row = t - w; row < t; ++row) {
                            const double* qr = q_all.data() + (size_t)row * m.dm + (size_t)qh * d;
                            ctx.window_queries.insert(ctx.window_queries.end(), qr, qr + d);
                            ctx.window_positions.push_back(row);
                        }
                    rep.scoring_ops += static_cast<int64_t>(ctx.window_positions.size()) * t * (d + 2);
                } else {
                    rep.scoring_ops += t;
                }
                ctx.keys = &keys_raw;
                ctx.scale = scale;
                auto mk = baseline_select(policy.select, ctx, budgets[(size_t)(l * H + kh)],
                                          derive_seed(seed, static_cast<uint64_t>(l), static_cast<uint64_t>(kh)));
                masks.insert(masks.end(), mk.begin(), mk.end());
            }
            Dev MK = up(masks);
            ck(lkv_cache_from_trace(&layer, MK.as<int32_t>(), t, &r, lws.ptr(), lws.bytes, stream()), "compaction");
            lws.status("prefill_with_eviction");
        }
        ws.status("prefill_with_eviction");
        select_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        KvCache part = ragged_to_cache(cfg, OF, LN, RK, RV, RP, H, d);
        for (int kh = 0; kh < H; ++kh) {
            const int idx = l * H + kh;
            cache.heads[(size_t)idx] = std::move(part.heads[(size_t)kh]);
            rep.retained_per_head[(size_t)idx] = cache.heads[(size_t)idx].retained();
            compressed += static_cast<int64_t>(cache.heads[(size_t)idx].retained()) * d * 2;
        }
        mlp_block(m, l, a, t);
    }
    ws.status("prefill_with_eviction");
    rep.evict_wall_seconds = select_seconds;
    MemoryModel mm;
    mm.n_layers = cfg.n_layers;
    mm.n_kv_heads = H;
    mm.head_dim = d;
    mm.bytes_per_element = 8.0;  // the reference's float64 accounting (evictsim.cpp:229)
    mm.tokens = t;
    const MemoryReport mr = kv_memory_bytes(mm, budgets);
    rep.kv_bytes_full = mr.full_bytes;
    rep.kv_bytes_compressed = mr.compressed_bytes;
    rep.reduction = mr.reduction_factor;
    return {std::move(cache), std::move(rep)};
}

// ============================ checkpoint.hpp ====================================================
namespace {
constexpr double kCkptVersion = 1.0;  // checkpoint.cpp:12

// container writer (container.cpp:45-76): u64 LE metadata length, compact JSON object of
// {"name": {"dtype": "f64", "shape": [...], "byte_offset": o, "byte_length": n}} in entry order,
// then the f64 payloads back to back
void write_container(const std::string& path, const std::vector<std::pair<std::string, const Tensor*>>& entries) {
    std::string meta = "{";
    uint64_t off = 0;
    for (size_t i = 0; i < entries.size(); ++i) {
        const Tensor& t = *entries[i].second;
        if (!t.defined()) throw contract_error("container: undefined tensor " + entries[i].first);
        for (size_t j = 0; j < i; ++j)
            if (entries[j].first == entries[i].first) throw contract_error("container: duplicate tensor name " + entries[i].first);
        std::string shape = "[";
        for (size_t d = 0; d < t.shape().size(); ++d) shape += (d ? "," : "") + std::to_string(t.shape()[d]);
        shape += "]";
        const uint64_t len = t.numel() * 8;
        meta += (i ? ",\"" : "\"") + entries[i].first + "\":{\"dtype\":\"f64\",\"shape\":" + shape +
                ",\"byte_offset\":" + std::to_string(off) + ",\"byte_length\":" + std::to_string(len) + "}";
        off += len;
    }
    meta += "}";
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw contract_error("container: cannot open for writing: " + path);
    unsigned char hdr[8];
    for (int i = 0; i < 8; ++i) hdr[i] = static_cast<unsigned char>((uint64_t)meta.size() >> (8 * i));
    bool ok = std::fwrite(hdr, 1, 8, f) == 8 && std::fwrite(meta.data(), 1, meta.size(), f) == meta.size();
    for (const auto& e : entries)
        ok = ok && std::fwrite(e.second->data(), 8, e.second->numel(), f) == e.second->numel();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw contract_error("container: write failed: " + path);
}

std::vector<std::pair<std::string, b200::ContainerTensor>> read(const std::string& path) {
    try {
        return b200::read_container(path);
    } catch (const b200::contract_error& e) {
        throw contract_error(std::string(e.what()).substr(10));  // same "contract: " taxonomy
    }
}
const b200::ContainerTensor& at(const std::vector<std::pair<std::string, b200::ContainerTensor>>& c,
                                const std::string& name) {
    for (const auto& e : c)
        if (e.first == name) return e.second;
    throw contract_error("container: missing tensor " + name);
}
}  // namespace

void save_model(const std::string& path, const ModelWeights& weights) {  // checkpoint.cpp:16-29
    const ModelConfig& c = weights.config;
    Tensor meta = make({9}, {kCkptVersion, (double)c.n_layers, (double)c.n_query_heads, (double)c.n_kv_heads,
                             (double)c.head_dim, (double)c.vocab_size, (double)c.max_seq_len, (double)c.mlp_hidden,
                             weights.frozen ? 1.0 : 0.0});
    std::vector<std::pair<std::string, const Tensor*>> e{{"__meta", &meta}};
    for (auto& nt : const_cast<ModelWeights&>(weights).named_params()) e.emplace_back(nt.first, nt.second);
    write_container(path, e);
}

ModelWeights load_model(const std::string& path) {  // checkpoint.cpp:31-52
    const auto c = read(path);
    const auto& meta = at(c, "__meta");
    if (meta.v.size() != 9 || meta.v[0] != kCkptVersion) throw contract_error("model checkpoint: unsupported metadata");
    ModelConfig cfg;
    cfg.n_layers = (int)meta.v[1];
    cfg.n_query_heads = (int)meta.v[2];
    cfg.n_kv_heads = (int)meta.v[3];
    cfg.head_dim = (int)meta.v[4];
    cfg.vocab_size = (int)meta.v[5];
    cfg.max_seq_len = (int)meta.v[6];
    cfg.mlp_hidden = (int)meta.v[7];
    ModelWeights w = init_model(cfg);
    for (auto& nt : w.named_params()) {
        const auto& t = at(c, nt.first);
        if (t.shape != nt.second->shape()) throw contract_error("model checkpoint: shape mismatch for " + nt.first);
        *nt.second = make(t.shape, t.v);
    }
    w.frozen = meta.v[8] != 0.0;
    return w;
}

void save_lkv_params(const std::string& path, const LkvParams& params) {  // checkpoint.cpp:54-65
    Tensor meta = make({5}, {kCkptVersion, (double)params.n_layers, (double)params.n_kv_heads, (double)params.d_e,
                             (double)params.d_head});
    std::vector<std::pair<std::string, const Tensor*>> e{{"__meta", &meta}};
    for (auto& nt : const_cast<LkvParams&>(params).named_params()) e.emplace_back(nt.first, nt.second);
    write_container(path, e);
}

LkvParams load_lkv_params(const std::string& path) {  // checkpoint.cpp:67-86
    const auto c = read(path);
    const auto& meta = at(c, "__meta");
    if (meta.v.size() != 5 || meta.v[0] != kCkptVersion) throw contract_error("policy checkpoint: unsupported metadata");
    ModelConfig cfg;
    cfg.n_layers = (int)meta.v[1];
    cfg.n_kv_heads = (int)meta.v[2];
    cfg.head_dim = (int)meta.v[4];
    cfg.n_query_heads = cfg.n_kv_heads;
    LkvParams p = init_lkv_params(cfg, 0, (int)meta.v[3]);
    for (auto& nt : p.named_params()) {
        const auto& t = at(c, nt.first);
        if (t.shape != nt.second->shape()) throw contract_error("policy checkpoint: shape mismatch for " + nt.first);
        *nt.second = make(t.shape, t.v);
    }
    return p;
}

}  // namespace lkv

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
