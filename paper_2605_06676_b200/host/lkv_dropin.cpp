// lkv_dropin.cpp -- C++ host layer: the reference's hot-path API (lkv::) re-expressed over
// the C ABI of the sm_100a kernels (include/lkv_b200.h).  See include/lkv_b200_dropin.hpp.
//
// Every call: validate like the reference (same exception types and conditions), upload
// host buffers, run the device kernels on a per-thread stream, synchronise, read back,
// and rethrow device-latched errors.  No computation happens on the host except the
// bookkeeping the reference itself does on the host (mask -> index lists, accounting).
#include "../../include/lkv_b200_dropin.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>

#include "../../include/lkv_b200.h"

namespace lkv::b200 {
namespace {

[[noreturn]] void rethrow(int status, const std::string& where) {
    const std::string msg = where + ": " + lkv_last_error();
    switch (status) {
        case LKV_ERR_CONTRACT: throw contract_error(msg);
        case LKV_ERR_NUMERIC: throw numeric_error(msg);
        case LKV_ERR_BUDGET: throw budget_error(msg);
        case LKV_ERR_OVERFLOW_GUARD: throw overflow_guard_error(msg);
        case LKV_ERR_DEGENERATE_MASK: throw degenerate_mask_error(msg);
        default: throw device_error(msg);
    }
}

void check(lkv_status s, const char* where) {
    if (s != LKV_OK) rethrow(s, where);
}

void cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw device_error(std::string(where) + ": " + cudaGetErrorString(e));
}

cudaStream_t stream() {
    thread_local cudaStream_t s = nullptr;
    if (!s) cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
    return s;
}

// RAII device buffer
struct Dev {
    void* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t bytes) : n(bytes) {
        if (bytes) cuda(cudaMalloc(&p, bytes + 256), "cudaMalloc");
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void* aligned() const { return reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)); }
};

template <class T>
Dev upload(const T* src, size_t count) {
    Dev d(sizeof(T) * count);
    if (count) cuda(cudaMemcpyAsync(d.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, stream()), "H2D");
    return d;
}

template <class T>
std::vector<T> download(const Dev& d, size_t count, size_t offset_elems = 0) {
    std::vector<T> out(count);
    if (count)
        cuda(cudaMemcpyAsync(out.data(), d.as<T>() + offset_elems, sizeof(T) * count, cudaMemcpyDeviceToHost, stream()),
             "D2H");
    cuda(cudaStreamSynchronize(stream()), "sync");
    return out;
}

// host fp64 -> device element (fp32 or bf16 bits, round to nearest even)
std::vector<uint16_t> to_bf16(std::span<const double> x) {
    std::vector<uint16_t> o(x.size());
    for (size_t i = 0; i < x.size(); ++i) o[i] = __bfloat16_as_ushort(__float2bfloat16_rn(static_cast<float>(x[i])));
    return o;
}
std::vector<float> to_f32(std::span<const double> x) { return std::vector<float>(x.begin(), x.end()); }

Dev upload_elems(std::span<const double> x, Precision prec) {
    if (prec == Precision::bf16) {
        auto v = to_bf16(x);
        return upload(v.data(), v.size());
    }
    auto v = to_f32(x);
    return upload(v.data(), v.size());
}

std::vector<double> download_elems(const Dev& d, size_t count, size_t offset_elems, Precision prec) {
    std::vector<double> out(count);
    if (prec == Precision::bf16) {
        auto v = download<uint16_t>(d, count, offset_elems);
        for (size_t i = 0; i < count; ++i) out[i] = __bfloat162float(__ushort_as_bfloat16(v[i]));
    } else {
        auto v = download<float>(d, count, offset_elems);
        for (size_t i = 0; i < count; ++i) out[i] = v[i];
    }
    return out;
}

int dtype_of(Precision p) { return p == Precision::bf16 ? LKV_BF16 : LKV_F32; }

struct Workspace {
    Dev buf;
    size_t bytes;
    explicit Workspace(size_t b) : buf(b + 256), bytes(b) {
        check(lkv_workspace_init(ptr(), bytes, (lkv_stream_t)stream()), "workspace");
    }
    void* ptr() const { return buf.aligned(); }
    void status(const char* where) { check(lkv_workspace_status(ptr(), (lkv_stream_t)stream()), where); }
};

// W1 [in x hidden] (reference layout) -> device W1^T [hidden x in] in the compute dtype
std::vector<double> transpose_w1(const Mlp2& m) {
    std::vector<double> t((size_t)m.in * m.hidden);
    for (int i = 0; i < m.in; ++i)
        for (int j = 0; j < m.hidden; ++j) t[(size_t)j * m.in + i] = m.w1[(size_t)i * m.hidden + j];
    return t;
}

void check_mlp(const Mlp2& m, int in) {
    if (m.in != in || m.hidden < 1 || m.w1.size() != (size_t)m.in * m.hidden || m.b1.size() != (size_t)m.hidden ||
        m.w2.size() != (size_t)m.hidden)
        throw contract_error("scorer shape does not match the key/value width");
}

}  // namespace

void require_b200() { check(lkv_device_check(), "device"); }

// ---- policy.cpp:110-129 -----------------------------------------------------------------------------
BudgetTable allocate_budgets(std::span<const double> scores, double target_ratio, int n_layers, int n_kv_heads) {
    if (!(target_ratio > 0.0 && target_ratio < 1.0)) throw budget_error("target ratio must lie in (0,1)");
    const int n = n_layers * n_kv_heads;
    if ((int)scores.size() != n || n < 1) throw contract_error("allocate_budgets: score length mismatch");
    Dev logits = upload(scores.data(), scores.size());
    Dev ratios(sizeof(double) * n), budgets(sizeof(int32_t) * n);
    Workspace ws(256);
    const int32_t one = 1;
    check(lkv_budgets(logits.as<double>(), n, target_ratio, LKV_BUDGET_FLOOR, &one, 1, 0, ratios.as<double>(),
                      budgets.as<int32_t>(), nullptr, ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "allocate_budgets");
    ws.status("allocate_budgets");
    BudgetTable t;
    t.n_layers = n_layers;
    t.n_kv_heads = n_kv_heads;
    t.target_ratio = target_ratio;
    t.ratios = download<double>(ratios, n);
    t.logits.assign(scores.begin(), scores.end());
    return t;
}

static std::vector<int> freeze(const BudgetTable& table, int t, int mode) {
    if (t < 1) throw contract_error("freeze_budgets: t must be >= 1");
    const int n = table.n_layers * table.n_kv_heads;
    if ((int)table.ratios.size() != n || n < 1) throw contract_error("freeze_budgets: ratio table size mismatch");
    Dev ratios = upload(table.ratios.data(), table.ratios.size());
    Dev budgets(sizeof(int32_t) * n);
    Workspace ws(256);
    const int32_t tt = t;
    check(lkv_freeze_budgets(ratios.as<double>(), n, table.target_ratio, mode, &tt, 1, 0, budgets.as<int32_t>(), nullptr,
                             ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "freeze_budgets");
    ws.status("freeze_budgets");
    auto b = download<int32_t>(budgets, n);
    return std::vector<int>(b.begin(), b.end());
}

std::vector<int> freeze_budgets(const BudgetTable& table, int t) { return freeze(table, t, LKV_BUDGET_FLOOR); }
std::vector<int> freeze_budgets_exact(const BudgetTable& table, int t) { return freeze(table, t, LKV_BUDGET_EXACT); }

// ---- policy.cpp:131-136 ------------------------------------------------------------------------------
std::vector<double> token_scores(std::span<const double> keys, std::span<const double> values, int t, int d,
                                 const Mlp2& scorer, Activation act, Precision prec) {
    if (t < 1 || d < 1 || keys.size() != (size_t)t * d) throw contract_error("token_scores: keys must be [t x d]");
    const bool kv = scorer.in == 2 * d;
    if (kv && values.size() != keys.size())
        throw contract_error("token_scores: keys/values must be rank-2 with equal first extents");
    check_mlp(scorer, kv ? 2 * d : d);
    for (double x : keys)
        if (!std::isfinite(x)) throw numeric_error("matmul: non-finite input");
    for (double x : values)
        if (!std::isfinite(x)) throw numeric_error("matmul: non-finite input");
    Dev K = upload_elems(keys, prec);
    Dev V = kv ? upload_elems(values, prec) : upload_elems(keys, prec);
    auto w1t = transpose_w1(scorer);
    Dev W1 = upload_elems(w1t, prec);
    auto b1 = to_f32(scorer.b1), w2 = to_f32(scorer.w2);
    Dev B1 = upload(b1.data(), b1.size()), W2 = upload(w2.data(), w2.size());
    Dev S(sizeof(float) * (size_t)t);
    const int32_t len = t;
    lkv_cache_desc c{1, 1, 1, d, t, dtype_of(prec), 0, K.p, V.p, &len};
    lkv_scorer_desc s{kv ? LKV_SCORER_KV : LKV_SCORER_K,
                      act == Activation::silu ? LKV_ACT_SILU : LKV_ACT_GELU_ERF,
                      scorer.hidden,
                      1,
                      0,
                      0,
                      W1.p,
                      B1.as<float>(),
                      W2.as<float>()};
    check(lkv_score(&c, &s, S.as<float>(), nullptr, 0, (lkv_stream_t)stream()), "token_scores");
    auto f = download<float>(S, t);
    return std::vector<double>(f.begin(), f.end());
}

// ---- soft_topk.cpp:191-201 / policy.cpp:152-154 ------------------------------------------------------
std::vector<int> hard_topk(std::span<const float> u, int b) {
    const int n = (int)u.size();
    if (b < 0 || b > n) throw budget_error("hard_topk: b outside [0, n]");
    std::vector<int> mask((size_t)n, 0);
    if (n == 0) return mask;
    Dev S = upload(u.data(), u.size());
    const int32_t len = n, bb = b;
    Dev Bd = upload(&bb, 1);
    lkv_cache_desc c{1, 1, 1, 8, n, LKV_F32, 0, nullptr, nullptr, &len};
    Dev offs(sizeof(int64_t) * 2), lens(sizeof(int32_t)), pos(sizeof(int32_t) * (size_t)(b > 0 ? b : 1));
    check(lkv_ragged_offsets(Bd.as<int32_t>(), 1, 0, offs.as<int64_t>(), (lkv_stream_t)stream()), "hard_topk");
    lkv_ragged_desc r{1, 8, LKV_F32, 0, b, offs.as<int64_t>(), lens.as<int32_t>(), nullptr, nullptr, pos.as<int32_t>()};
    Workspace ws(lkv_workspace_bytes(&c, 1));
    check(lkv_select(&c, S.as<float>(), Bd.as<int32_t>(), &r, 0, ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "hard_topk");
    ws.status("hard_topk");
    for (int32_t p : download<int32_t>(pos, (size_t)b)) mask[(size_t)p] = 1;
    return mask;
}

std::vector<int> inference_select(std::span<const float> u, int b) { return hard_topk(u, b); }

// ---- shared upload of a dense trace ----------------------------------------------------------------------
namespace {
struct DenseUpload {
    Dev K, V;
    int32_t len;
    lkv_cache_desc desc;
};

DenseUpload upload_trace(const KvTrace& tr, Precision prec) {
    const int heads = tr.n_layers * tr.n_kv_heads;
    if (tr.t < 1 || tr.head_dim < 1 || (int)tr.keys.size() != heads || (int)tr.values.size() != heads)
        throw contract_error("trace head count mismatch");
    std::vector<double> k((size_t)heads * tr.t * tr.head_dim), v(k.size());
    for (int h = 0; h < heads; ++h) {
        if (tr.keys[(size_t)h].size() != (size_t)tr.t * tr.head_dim || tr.values[(size_t)h].size() != (size_t)tr.t * tr.head_dim)
            throw contract_error("trace head must be [t x head_dim]");
        std::memcpy(k.data() + (size_t)h * tr.t * tr.head_dim, tr.keys[(size_t)h].data(), sizeof(double) * tr.t * tr.head_dim);
        std::memcpy(v.data() + (size_t)h * tr.t * tr.head_dim, tr.values[(size_t)h].data(), sizeof(double) * tr.t * tr.head_dim);
    }
    DenseUpload u{upload_elems(k, prec), upload_elems(v, prec), tr.t, {}};
    u.desc = lkv_cache_desc{1, tr.n_layers, tr.n_kv_heads, tr.head_dim, tr.t, dtype_of(prec), 0, u.K.p, u.V.p, &u.len};
    return u;
}

KvCache download_ragged(const KvTrace& tr, const Dev& offs, const Dev& lens, const Dev& rk, const Dev& rv,
                        const Dev& rp, Precision prec) {
    const int heads = tr.n_layers * tr.n_kv_heads;
    auto o = download<int64_t>(offs, (size_t)heads + 1);
    auto l = download<int32_t>(lens, (size_t)heads);
    KvCache cache;
    cache.n_layers = tr.n_layers;
    cache.n_kv_heads = tr.n_kv_heads;
    cache.head_dim = tr.head_dim;
    cache.tokens_seen = tr.t;
    cache.heads.resize((size_t)heads);
    for (int h = 0; h < heads; ++h) {
        HeadCache& hc = cache.heads[(size_t)h];
        const size_t rows = (size_t)l[(size_t)h];
        hc.keys = download_elems(rk, rows * tr.head_dim, (size_t)o[(size_t)h] * tr.head_dim, prec);
        hc.values = download_elems(rv, rows * tr.head_dim, (size_t)o[(size_t)h] * tr.head_dim, prec);
        auto p = download<int32_t>(rp, rows, (size_t)o[(size_t)h]);
        hc.retained_positions.assign(p.begin(), p.end());
    }
    return cache;
}

size_t esize(Precision p) { return p == Precision::bf16 ? 2 : 4; }
}  // namespace

// ---- model.cpp:289-315 ----------------------------------------------------------------------------------
KvCache cache_from_trace(const KvTrace& tr, const std::vector<std::vector<int>>& hard_masks, Precision prec) {
    const int heads = tr.n_layers * tr.n_kv_heads;
    if ((int)hard_masks.size() != heads) throw contract_error("cache_from_trace: one mask per head required");
    std::vector<int32_t> masks((size_t)heads * tr.t);
    for (int h = 0; h < heads; ++h) {
        const auto& m = hard_masks[(size_t)h];
        if ((int)m.size() != tr.t) throw contract_error("cache_from_trace: mask length mismatch");
        std::copy(m.begin(), m.end(), masks.begin() + (size_t)h * tr.t);
    }
    DenseUpload du = upload_trace(tr, prec);
    Dev M = upload(masks.data(), masks.size());
    Workspace ws(lkv_workspace_bytes(&du.desc, 1));
    // device mask scan: counts size the ragged cache, then compaction + 16-byte row gather
    Dev cnt(sizeof(int32_t) * (size_t)heads);
    check(lkv_mask_counts(&du.desc, M.as<int32_t>(), tr.t, cnt.as<int32_t>(), ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "cache_from_trace");
    int64_t rows = 0;
    for (int32_t c : download<int32_t>(cnt, (size_t)heads)) rows += c;
    Dev offs(sizeof(int64_t) * ((size_t)heads + 1));
    Dev lens(sizeof(int32_t) * (size_t)heads);
    Dev rp(sizeof(int32_t) * (size_t)(rows ? rows : 1));
    Dev rk(esize(prec) * (size_t)(rows ? rows : 1) * tr.head_dim), rv(esize(prec) * (size_t)(rows ? rows : 1) * tr.head_dim);
    lkv_ragged_desc r{heads, tr.head_dim, dtype_of(prec), 0, rows, offs.as<int64_t>(), lens.as<int32_t>(), rk.p, rv.p,
                      rp.as<int32_t>()};
    check(lkv_cache_from_trace(&du.desc, M.as<int32_t>(), tr.t, &r, ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "cache_from_trace");
    ws.status("cache_from_trace");
    return download_ragged(tr, offs, lens, rk, rv, rp, prec);
}

// ---- evictsim.cpp:95-238 (K/V-given form) ----------------------------------------------------------------
std::pair<KvCache, SimReport> prefill_with_eviction(const KvTrace& tr, const std::vector<int>& budgets,
                                                    const std::vector<Mlp2>& scorers, Activation act,
                                                    Precision prec) {
    const int heads = tr.n_layers * tr.n_kv_heads;
    if ((int)budgets.size() != heads) throw contract_error("prefill_with_eviction: one budget per head required");
    for (int b : budgets)
        if (b < 0 || b > tr.t) throw budget_error("prefill_with_eviction: budget outside [0, t]");
    const bool per_head = (int)scorers.size() == heads;
    if (!per_head && (int)scorers.size() != tr.n_layers)
        throw contract_error("prefill_with_eviction: one scorer per (layer, head) or per layer required");
    const int hidden = scorers.front().hidden;
    const int in = scorers.front().in;
    if (in != tr.head_dim && in != 2 * tr.head_dim) throw contract_error("scorer input must be d or 2d");
    std::vector<double> w1t, b1, w2;
    for (const Mlp2& m : scorers) {
        check_mlp(m, in);
        if (m.hidden != hidden) throw contract_error("all scorers must share one hidden width");
        auto t = transpose_w1(m);
        w1t.insert(w1t.end(), t.begin(), t.end());
        b1.insert(b1.end(), m.b1.begin(), m.b1.end());
        w2.insert(w2.end(), m.w2.begin(), m.w2.end());
    }
    DenseUpload du = upload_trace(tr, prec);
    Dev W1 = upload_elems(w1t, prec);
    auto b1f = to_f32(b1), w2f = to_f32(w2);
    Dev B1 = upload(b1f.data(), b1f.size()), W2 = upload(w2f.data(), w2f.size());
    lkv_scorer_desc sd{in == tr.head_dim ? LKV_SCORER_K : LKV_SCORER_KV,
                       act == Activation::silu ? LKV_ACT_SILU : LKV_ACT_GELU_ERF,
                       hidden,
                       (int)scorers.size(),
                       per_head ? tr.n_kv_heads : 1,
                       per_head ? 1 : 0,
                       W1.p,
                       B1.as<float>(),
                       W2.as<float>()};
    std::vector<int32_t> b32(budgets.begin(), budgets.end());
    int64_t rows = 0;
    for (int b : budgets) rows += b;
    Dev Bd = upload(b32.data(), b32.size());
    Dev offs(sizeof(int64_t) * ((size_t)heads + 1)), lens(sizeof(int32_t) * heads);
    Dev rk(esize(prec) * (size_t)(rows ? rows : 1) * tr.head_dim), rv(esize(prec) * (size_t)(rows ? rows : 1) * tr.head_dim);
    Dev rp(sizeof(int32_t) * (size_t)(rows ? rows : 1));
    Dev S(sizeof(float) * (size_t)heads * tr.t);
    lkv_ragged_desc r{heads, tr.head_dim, dtype_of(prec), 0, rows, offs.as<int64_t>(), lens.as<int32_t>(), rk.p, rv.p,
                      rp.as<int32_t>()};
    Workspace ws(lkv_workspace_bytes(&du.desc, heads));
    cudaEvent_t e0, e1;
    cuda(cudaEventCreate(&e0), "event");
    cuda(cudaEventCreate(&e1), "event");
    cuda(cudaEventRecord(e0, stream()), "event");
    check(lkv_ragged_offsets(Bd.as<int32_t>(), heads, 0, offs.as<int64_t>(), (lkv_stream_t)stream()), "prefill");
    check(lkv_score(&du.desc, &sd, S.as<float>(), nullptr, 0, (lkv_stream_t)stream()), "prefill score");
    check(lkv_select(&du.desc, S.as<float>(), Bd.as<int32_t>(), &r, 1, ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "prefill select");
    cuda(cudaEventRecord(e1, stream()), "event");
    ws.status("prefill_with_eviction");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::pair<KvCache, SimReport> out{download_ragged(tr, offs, lens, rk, rv, rp, prec), SimReport{}};
    SimReport& rep = out.second;
    rep.retained_per_head.resize((size_t)heads);
    for (int h = 0; h < heads; ++h) rep.retained_per_head[(size_t)h] = out.first.heads[(size_t)h].retained();
    rep.evict_device_seconds = ms * 1e-3;
    rep.scoring_ops = (int64_t)heads * tr.t * ((int64_t)in * hidden + 3 * hidden);  // evictsim.cpp:172
    MemoryModel mm;
    mm.n_layers = tr.n_layers;
    mm.n_kv_heads = tr.n_kv_heads;
    mm.head_dim = tr.head_dim;
    mm.bytes_per_element = 8.0;  // fp64 host storage, as evictsim.cpp:231
    mm.tokens = tr.t;
    const MemoryReport mr = kv_memory_bytes(mm, budgets);
    rep.kv_bytes_full = mr.full_bytes;
    rep.kv_bytes_compressed = mr.compressed_bytes;
    rep.reduction = mr.reduction_factor;
    return out;
}

// ---- model.cpp:240-265 ------------------------------------------------------------------------------------
std::vector<double> decode_attention(KvCache& cache, std::span<const double> q, int n_q_heads,
                                     std::span<const double> k_new, std::span<const double> v_new, Precision prec) {
    const int L = cache.n_layers, H = cache.n_kv_heads, d = cache.head_dim;
    if (L < 1 || H < 1 || d < 1 || (int)cache.heads.size() != L * H) throw contract_error("decode_step: cache head count mismatch");
    if (n_q_heads < H || n_q_heads % H) throw contract_error("decode_step: n_q_heads must be a multiple of n_kv_heads");
    if (q.size() != (size_t)L * n_q_heads * d || k_new.size() != (size_t)L * H * d || v_new.size() != k_new.size())
        throw contract_error("decode_step: q [L][Hq][d], k/v [L][H][d] required");
    const int heads = L * H;
    std::vector<int32_t> lens((size_t)heads), pos;
    std::vector<double> k, v;
    std::vector<int64_t> offs((size_t)heads + 1, 0);
    for (int h = 0; h < heads; ++h) {
        const HeadCache& hc = cache.heads[(size_t)h];
        lens[(size_t)h] = hc.retained();
        offs[(size_t)h + 1] = offs[(size_t)h] + hc.retained() + 1;  // one row of decode slack
        k.insert(k.end(), hc.keys.begin(), hc.keys.end());
        v.insert(v.end(), hc.values.begin(), hc.values.end());
        k.insert(k.end(), (size_t)d, 0.0);
        v.insert(v.end(), (size_t)d, 0.0);
        pos.insert(pos.end(), hc.retained_positions.begin(), hc.retained_positions.end());
        pos.push_back(-1);
    }
    const int64_t rows = offs.back();
    Dev K = upload_elems(k, prec), V = upload_elems(v, prec);
    Dev P = upload(pos.data(), pos.size()), Ld = upload(lens.data(), lens.size()), O = upload(offs.data(), offs.size());
    Dev Q = upload_elems(q, prec), NK = upload_elems(k_new, prec), NV = upload_elems(v_new, prec);
    const int32_t seen = cache.tokens_seen;
    Dev TS = upload(&seen, 1);
    Dev OUT(esize(prec) * q.size());
    lkv_ragged_desc r{heads, d, dtype_of(prec), 1, rows, O.as<int64_t>(), Ld.as<int32_t>(), K.p, V.p, P.as<int32_t>()};
    Workspace ws(lkv_decode_workspace_bytes(&r, n_q_heads / H));
    check(lkv_decode_plan(&r, ws.ptr(), ws.bytes, (lkv_stream_t)stream()), "decode plan");
    check(lkv_decode_step(&r, 1, L, H, n_q_heads, Q.p, NK.p, NV.p, TS.as<int32_t>(), OUT.p, 1.0 / std::sqrt((double)d),
                          ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "decode_step");
    ws.status("decode_step");
    auto out = download_elems(OUT, q.size(), 0, prec);
    // the reference appends the new k, v and position to every head (model.cpp:240-248)
    for (int h = 0; h < heads; ++h) {
        HeadCache& hc = cache.heads[(size_t)h];
        hc.keys.insert(hc.keys.end(), k_new.begin() + (size_t)h * d, k_new.begin() + (size_t)(h + 1) * d);
        hc.values.insert(hc.values.end(), v_new.begin() + (size_t)h * d, v_new.begin() + (size_t)(h + 1) * d);
        hc.retained_positions.push_back(cache.tokens_seen);
    }
    cache.tokens_seen += 1;
    return out;
}

std::string budget_table_csv(const BudgetTable& table) {  // policy.cpp:301-311
    std::string out = "layer,head,ratio\n";
    char buf[64];
    for (int l = 0; l < table.n_layers; ++l)
        for (int h = 0; h < table.n_kv_heads; ++h) {
            std::snprintf(buf, sizeof buf, "%d,%d,%.6f\n", l, h, table.at(l, h));
            out += buf;
        }
    return out;
}

// ---- soft_topk.cpp:111-189 (training) ---------------------------------------------------
static SoftTopKOutput soft_topk_impl(std::span<const double> x, double k, double tau, std::span<const double> noise,
                                     double noise_scale) {
    if (!(tau > 0.0)) throw contract_error("soft_topk_forward: tau must be positive");  // soft_topk.cpp:112
    const int n = (int)x.size();
    if (n < 1) throw contract_error("soft_topk_forward: empty scores");  // :114
    Dev X = upload(x.data(), x.size()), K = upload(&k, 1);
    Dev N = noise.empty() ? Dev() : upload(noise.data(), noise.size());
    if (!noise.empty() && (int)noise.size() != n) throw contract_error("training_mask: noise length must equal t");
    Dev VAL(sizeof(double) * n), DEN(sizeof(double) * n), LAM(sizeof(double));
    Workspace ws(256);
    check(lkv_soft_topk_fwd(X.as<double>(), noise.empty() ? nullptr : N.as<double>(), noise_scale, 1, n, n,
                            K.as<double>(), tau, VAL.as<double>(), DEN.as<double>(), nullptr, LAM.as<double>(), ws.ptr(),
                            ws.bytes, (lkv_stream_t)stream()),
          "soft_topk_forward");
    ws.status("soft_topk_forward");
    SoftTopKOutput out;
    out.values = download<double>(VAL, n);
    out.density_terms = download<double>(DEN, n);
    out.threshold_lambda = download<double>(LAM, 1)[0];
    const double eps = std::min(1e-3, 0.01 * n);  // clamp_budget (soft_topk.cpp:27-33)
    out.clamped_k = std::min(std::max(k, eps), n - eps);
    out.tau = tau;
    return out;
}

SoftTopKOutput soft_topk_forward(std::span<const double> x, double k, double tau) {
    return soft_topk_impl(x, k, tau, {}, 0.0);
}

SoftTopKOutput training_mask(std::span<const double> u, double b_continuous, double tau,
                             std::span<const double> gumbel_noise, double noise_scale) {
    return soft_topk_impl(u, b_continuous, tau, gumbel_noise, noise_scale);
}

std::pair<std::vector<double>, double> soft_topk_vjp(const SoftTopKOutput& saved, std::span<const double> upstream,
                                                     double tau) {
    const size_t n = saved.values.size();
    if (upstream.size() != n) throw contract_error("soft_topk_vjp: upstream length mismatch");  // :170
    if (!(tau > 0.0)) throw contract_error("soft_topk_vjp: tau must be positive");             // :171
    Dev D = upload(saved.density_terms.data(), n), U = upload(upstream.data(), n);
    Dev GX(sizeof(double) * n), GK(sizeof(double));
    check(lkv_soft_topk_vjp(D.as<double>(), U.as<double>(), 1, (int)n, (int64_t)n, tau, GX.as<double>(), GK.as<double>(),
                            (lkv_stream_t)stream()),
          "soft_topk_vjp");
    return {download<double>(GX, n), download<double>(GK, 1)[0]};
}

// ---- attention.cpp:46-201 (training) ---------------------------------------------------
static lkv_attn_desc attn_desc(const AttentionCall& c, Precision prec) {
    if (c.n_q < 1 || c.t < 1 || c.d < 1) throw contract_error("attention: empty extents");  // attention.cpp:34
    if (c.queries.size() != (size_t)c.n_q * c.d) throw contract_error("attention: query size");
    if (c.keys.size() != (size_t)c.t * c.d) throw contract_error("attention: key size");
    if (c.values.size() != (size_t)c.t * c.d) throw contract_error("attention: value size");
    if (!c.soft_mask.empty() && c.soft_mask.size() != (size_t)c.t) throw contract_error("attention: mask length must equal t");
    return lkv_attn_desc{1, 1, 1, c.n_q, c.t, c.d, dtype_of(prec), c.causal ? 1 : 0, c.query_pos_offset,
                         c.self_always_retained ? 1 : 0, c.scale};
}

std::vector<double> masked_attention_dense(const AttentionCall& call, AttentionSaved* saved, Precision prec) {
    lkv_attn_desc a = attn_desc(call, prec);
    Dev Q = upload_elems(call.queries, prec), K = upload_elems(call.keys, prec), V = upload_elems(call.values, prec);
    std::vector<float> m(call.soft_mask.begin(), call.soft_mask.end());
    Dev M = m.empty() ? Dev() : upload(m.data(), m.size());
    Dev OUT(esize(prec) * call.queries.size()), LSE(sizeof(float) * call.n_q);
    const size_t wsb = lkv_attn_workspace_bytes(&a);
    if (wsb == 0) check(lkv_masked_attention_fwd(&a, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr),
                        "masked_attention_dense");
    Workspace ws(wsb);
    check(lkv_masked_attention_fwd(&a, Q.p, K.p, V.p, m.empty() ? nullptr : M.as<float>(), OUT.p, LSE.as<float>(), ws.ptr(),
                                   ws.bytes, (lkv_stream_t)stream()),
          "masked_attention_dense");
    ws.status("masked_attention_dense");
    auto out = download_elems(OUT, call.queries.size(), 0, prec);
    if (saved) {
        saved->lse = download<float>(LSE, call.n_q);
        saved->out = out;
        saved->prec = prec;
    }
    return out;
}

AttentionGrads masked_attention_vjp(const AttentionCall& call, const AttentionSaved& saved,
                                    const std::vector<double>& upstream) {
    const Precision prec = saved.prec;
    lkv_attn_desc a = attn_desc(call, prec);
    if (upstream.size() != (size_t)call.n_q * call.d) throw contract_error("attention vjp: upstream size");
    if (saved.lse.size() != (size_t)call.n_q || saved.out.size() != upstream.size())
        throw contract_error("attention vjp: stale saved state");
    Dev Q = upload_elems(call.queries, prec), K = upload_elems(call.keys, prec), V = upload_elems(call.values, prec);
    std::vector<float> m(call.soft_mask.begin(), call.soft_mask.end());
    Dev M = m.empty() ? Dev() : upload(m.data(), m.size());
    Dev O = upload_elems(saved.out, prec), U = upload_elems(upstream, prec), LSE = upload(saved.lse.data(), saved.lse.size());
    Dev DQ(sizeof(float) * call.queries.size()), DK(sizeof(float) * call.keys.size()), DV(sizeof(float) * call.values.size());
    Dev DM(sizeof(float) * (m.empty() ? 1 : m.size()));
    Workspace ws(lkv_attn_workspace_bytes(&a));
    check(lkv_masked_attention_bwd(&a, Q.p, K.p, V.p, m.empty() ? nullptr : M.as<float>(), O.p, LSE.as<float>(), U.p,
                                   DQ.as<float>(), DK.as<float>(), DV.as<float>(), m.empty() ? nullptr : DM.as<float>(),
                                   ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "masked_attention_vjp");
    ws.status("masked_attention_vjp");
    auto widen = [](const std::vector<float>& f) { return std::vector<double>(f.begin(), f.end()); };
    AttentionGrads g;
    g.queries = widen(download<float>(DQ, call.queries.size()));
    g.keys = widen(download<float>(DK, call.keys.size()));
    g.values = widen(download<float>(DV, call.values.size()));
    if (!m.empty()) g.soft_mask = widen(download<float>(DM, m.size()));
    return g;
}

// ---- checkpoint.cpp:68-86 / container.cpp:92-137 --------------------------------------------------------
namespace {
// Just enough JSON for the container metadata: an ordered object of objects holding
// strings, non-negative integers and arrays of integers.
struct MetaRec {
    std::string name, dtype;
    std::vector<int> shape;
    uint64_t off = 0, len = 0;
};
struct JsonCursor {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
    }
    void expect(char c) {
        ws();
        if (i >= s.size() || s[i] != c) throw contract_error("container: bad metadata JSON");
        ++i;
    }
    bool peek(char c) {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string str() {
        expect('"');
        std::string o;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') ++i;
            if (i < s.size()) o += s[i++];
        }
        expect('"');
        return o;
    }
    uint64_t num() {
        ws();
        uint64_t v = 0;
        size_t j = i;
        while (i < s.size() && s[i] >= '0' && s[i] <= '9') v = v * 10 + (uint64_t)(s[i++] - '0');
        if (i == j) throw contract_error("container: bad metadata JSON");
        return v;
    }
};

std::vector<MetaRec> parse_meta(const std::string& js) {
    JsonCursor c{js};
    std::vector<MetaRec> out;
    c.expect('{');
    while (!c.peek('}')) {
        MetaRec r;
        r.name = c.str();
        c.expect(':');
        c.expect('{');
        int seen = 0;
        while (!c.peek('}')) {
            const std::string key = c.str();
            c.expect(':');
            if (key == "dtype") {
                r.dtype = c.str();
                seen |= 1;
            } else if (key == "shape") {
                c.expect('[');
                while (!c.peek(']')) {
                    r.shape.push_back((int)c.num());
                    if (c.peek(',')) c.expect(',');
                }
                c.expect(']');
                seen |= 2;
            } else if (key == "byte_offset") {
                r.off = c.num();
                seen |= 4;
            } else if (key == "byte_length") {
                r.len = c.num();
                seen |= 8;
            } else {
                throw contract_error("container: unexpected field " + key);
            }
            if (c.peek(',')) c.expect(',');
        }
        c.expect('}');
        if (seen != 15) throw contract_error("container: incomplete record for " + r.name);
        out.push_back(r);
        if (c.peek(',')) c.expect(',');
    }
    c.expect('}');
    return out;
}

using Loaded = ContainerTensor;
}  // namespace

std::vector<std::pair<std::string, ContainerTensor>> read_container(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw contract_error("container: cannot open: " + path);
    std::string raw;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) raw.append(buf, got);
    std::fclose(f);
    if (raw.size() < 8) throw contract_error("container: truncated header");
    uint64_t meta_len = 0;
    for (int i = 0; i < 8; ++i) meta_len |= (uint64_t)(unsigned char)raw[(size_t)i] << (8 * i);
    if (8 + meta_len > raw.size()) throw contract_error("container: truncated metadata");
    const auto recs = parse_meta(raw.substr(8, meta_len));
    const char* payload = raw.data() + 8 + meta_len;
    const uint64_t payload_size = raw.size() - 8 - meta_len;
    std::vector<std::pair<std::string, Loaded>> out;
    uint64_t expected = 0;
    for (const MetaRec& r : recs) {
        const size_t es = r.dtype == "f64" ? 8 : r.dtype == "f32" ? 4 : 0;
        if (!es) throw contract_error("container: unknown dtype " + r.dtype);
        if (r.off != expected) throw contract_error("container: offsets must be contiguous and in order");
        if (r.off + r.len > payload_size) throw contract_error("container: payload shorter than metadata claims");
        size_t numel = 1;
        for (int d : r.shape) numel *= (size_t)d;
        if (r.len != numel * es) throw contract_error("container: byte length mismatch for " + r.name);
        Loaded L{r.shape, std::vector<double>(numel)};
        if (es == 8) {
            std::memcpy(L.v.data(), payload + r.off, r.len);
        } else {
            std::vector<float> tmp(numel);
            std::memcpy(tmp.data(), payload + r.off, r.len);
            for (size_t i = 0; i < numel; ++i) L.v[i] = tmp[i];
        }
        out.emplace_back(r.name, std::move(L));
        expected = r.off + r.len;
    }
    if (expected != payload_size) throw contract_error("container: trailing bytes after last tensor");
    return out;
}

namespace {
const Loaded& entry(const std::vector<std::pair<std::string, Loaded>>& c, const std::string& name) {
    for (const auto& e : c)
        if (e.first == name) return e.second;
    throw contract_error("container: missing tensor " + name);
}

Mlp2 mlp_of(const std::vector<std::pair<std::string, Loaded>>& c, const std::string& p, int in, int hidden) {
    const Loaded &w1 = entry(c, p + "w1"), &b1 = entry(c, p + "b1"), &w2 = entry(c, p + "w2");
    if (w1.shape != std::vector<int>{in, hidden} || b1.shape != std::vector<int>{hidden} ||
        w2.shape != std::vector<int>{hidden, 1})
        throw contract_error("policy checkpoint: shape mismatch for " + p);
    return Mlp2{in, hidden, w1.v, b1.v, w2.v};
}
}  // namespace

LkvParams load_lkv_params(const std::string& path) {
    const auto c = read_container(path);
    const Loaded& meta = entry(c, "__meta");
    if (meta.v.size() != 5 || meta.v[0] != 1.0) throw contract_error("policy checkpoint: unsupported metadata");
    LkvParams p;
    p.n_layers = (int)meta.v[1];
    p.n_kv_heads = (int)meta.v[2];
    p.d_e = (int)meta.v[3];
    p.d_head = (int)meta.v[4];
    const int n = p.n_layers * p.n_kv_heads;
    const Loaded& emb = entry(c, "head_embeddings");
    if (emb.shape != std::vector<int>{n, p.d_e}) throw contract_error("policy checkpoint: shape mismatch for head_embeddings");
    p.head_embeddings = emb.v;
    p.head_predictor = mlp_of(c, "head_predictor.", p.d_e, p.d_e / 2);
    for (int i = 0; i < n; ++i)
        p.token_scorers.push_back(mlp_of(c, "token_scorers." + std::to_string(i) + ".", 2 * p.d_head, p.d_head));
    return p;
}

std::vector<double> head_scores(const LkvParams& p) {  // policy.cpp:106-108 on the device (fp64 scorer)
    const int n = p.n_layers * p.n_kv_heads, de = p.d_e, hid = p.head_predictor.hidden;
    if ((int)p.head_embeddings.size() != n * de) throw contract_error("head_scores: embedding table size mismatch");
    Dev E = upload(p.head_embeddings.data(), p.head_embeddings.size());
    Dev W1 = upload(p.head_predictor.w1.data(), p.head_predictor.w1.size());
    Dev B1 = upload(p.head_predictor.b1.data(), p.head_predictor.b1.size());
    Dev W2 = upload(p.head_predictor.w2.data(), p.head_predictor.w2.size());
    Dev U(sizeof(double) * (size_t)n);
    Workspace ws(256);
    check(lkv_f64_token_scores(n, de, LKV_SCORER_K, E.as<double>(), de, nullptr, 0, W1.as<double>(), B1.as<double>(),
                               W2.as<double>(), hid, LKV_ACT_SILU, U.as<double>(), ws.ptr(), ws.bytes, (lkv_stream_t)stream()),
          "head_scores");
    ws.status("head_scores");
    return download<double>(U, (size_t)n);
}

// ---- evictsim.cpp:56-81 (accounting) ------------------------------------------------------------------------
MemoryReport kv_memory_bytes(const MemoryModel& m, double retention) {
    if (m.n_layers < 1 || m.n_kv_heads < 1 || m.head_dim < 1 || m.tokens < 1 || !(m.bytes_per_element > 0.0))
        throw contract_error("memory model: all extents must be positive");
    if (!(retention > 0.0) || retention > 1.0) throw budget_error("kv_memory_bytes: retention must lie in (0, 1]");
    MemoryReport r;
    r.full_bytes = (double)m.n_layers * m.n_kv_heads * m.head_dim * 2.0 * m.bytes_per_element * (double)m.tokens;
    r.compressed_bytes = retention * r.full_bytes;
    r.reduction_factor = r.full_bytes / r.compressed_bytes;
    return r;
}

MemoryReport kv_memory_bytes(const MemoryModel& m, const std::vector<int>& per_head_budgets) {
    if (m.n_layers < 1 || m.n_kv_heads < 1 || m.head_dim < 1 || m.tokens < 1 || !(m.bytes_per_element > 0.0))
        throw contract_error("memory model: all extents must be positive");
    if ((int)per_head_budgets.size() != m.n_layers * m.n_kv_heads)
        throw contract_error("kv_memory_bytes: one budget per head required");
    MemoryReport r;
    r.full_bytes = (double)m.n_layers * m.n_kv_heads * m.head_dim * 2.0 * m.bytes_per_element * (double)m.tokens;
    double kept = 0.0;
    for (int b : per_head_budgets) kept += (double)b;
    r.compressed_bytes = kept * m.head_dim * 2.0 * m.bytes_per_element;
    r.reduction_factor = r.compressed_bytes > 0.0 ? r.full_bytes / r.compressed_bytes
                                                  : std::numeric_limits<double>::infinity();
    return r;
}

}  // namespace lkv::b200
