// c_api.cu -- the extern "C" drop-in boundary (include/lkv_b200.h).
//
// Host-side validation mirrors the reference's exception behaviour (budget /
// contract / numeric errors, errors.hpp:10-32); device-side failures are
// latched into the caller's workspace.  No allocation of caller memory, no
// CPU fallback: every compute entry point launches sm_100a kernels or fails.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lkv_b200.h"
#include "kernels.cuh"


using namespace lkv_dev;

namespace {
thread_local std::string g_err;
}  // namespace

// shared with comm.cu
lkv_status lkv_internal_fail(lkv_status code, const std::string& msg) {
    g_err = msg;
    return code;
}

namespace {

lkv_status fail(lkv_status code, const std::string& msg) { return lkv_internal_fail(code, msg); }

lkv_status cuda_fail(cudaError_t e, const char* where) {
    return fail(LKV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LKV_CUDA(call, where)                            \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

int elem_bytes(int dtype) { return dtype == LKV_F64 ? 8 : dtype == LKV_F32 ? 4 : 2; }

int num_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// Non-blocking helper streams per (host thread, device) for fork/join inside a call:
// `side` runs the latency-bound LKV-H solve, `copy` the host<->device transfers.
cudaStream_t helper_stream(int which) {
    thread_local cudaStream_t streams[3][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    cudaStream_t& s = streams[which][dev];
    if (!s && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    return s;
}
cudaStream_t side_stream() { return helper_stream(0); }
cudaStream_t copy_stream() { return helper_stream(1); }
cudaStream_t d2h_stream() { return helper_stream(2); }  // device->host, so it overlaps H2D (full duplex)

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// ---- TMA descriptor encoding (driver entry point, no -lcuda) ----------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 tensor [rows][inner] (row-major), box = 64 x box_rows, 128-byte swizzle.
lkv_status make_map_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(LKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(LKV_ERR_CONTRACT, "TMA base must be 16-byte aligned");
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LKV_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LKV_OK;
}

// ---- descriptor validation ---------------------------------------------------------------------
lkv_status check_cache(const lkv_cache_desc* c, bool need_kv) {
    if (!c) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    if (c->n_seq < 1 || c->n_seq > LKV_MAX_SEQ) return fail(LKV_ERR_CONTRACT, "n_seq must lie in [1, LKV_MAX_SEQ]");
    if (c->n_layers < 1 || c->n_kv_heads < 1) return fail(LKV_ERR_CONTRACT, "n_layers and n_kv_heads must be >= 1");
    if (c->head_dim < 8 || c->head_dim % 8) return fail(LKV_ERR_CONTRACT, "head_dim must be a positive multiple of 8");
    {
        const int units = c->head_dim * elem_bytes(c->dtype) / 16;
        if (units & (units - 1)) return fail(LKV_ERR_UNSUPPORTED, "row bytes must be a power-of-two multiple of 16");
    }
    if (c->dtype != LKV_F32 && c->dtype != LKV_BF16 && c->dtype != LKV_F64) return fail(LKV_ERR_CONTRACT, "unknown dtype");
    if (c->max_tokens < 1) return fail(LKV_ERR_CONTRACT, "max_tokens must be >= 1");
    if (!c->seq_lens) return fail(LKV_ERR_CONTRACT, "seq_lens (host) is null");
    for (int s = 0; s < c->n_seq; ++s)
        if (c->seq_lens[s] < 1 || c->seq_lens[s] > c->max_tokens)
            return fail(LKV_ERR_CONTRACT, "seq_lens[s] must lie in [1, max_tokens]");
    const int64_t heads = (int64_t)c->n_seq * c->n_layers * c->n_kv_heads;
    if (heads * c->max_tokens >= (int64_t(1) << 31)) return fail(LKV_ERR_CONTRACT, "cache rows exceed 2^31");
    if (need_kv && (!c->keys || !c->values)) return fail(LKV_ERR_CONTRACT, "keys/values are null");
    return LKV_OK;
}

SeqTable make_seq(const lkv_cache_desc* c) {
    SeqTable s;
    memset(&s, 0, sizeof s);
    s.n_seq = c->n_seq;
    s.n_layers = c->n_layers;
    s.n_kv_heads = c->n_kv_heads;
    s.head_dim = c->head_dim;
    s.T = c->max_tokens;
    for (int i = 0; i < c->n_seq; ++i) s.len[i] = c->seq_lens[i];
    return s;
}

int64_t n_heads_of(const lkv_cache_desc* c) { return (int64_t)c->n_seq * c->n_layers * c->n_kv_heads; }

// ---- workspace layout -----------------------------------------------------------------------------
struct EvictWs {
    size_t err, ratios, budgets, budgets_all, scores, hist, state, chunk_out, chunk_eqb, cands, total;
};

EvictWs evict_layout(const lkv_cache_desc* c, int n_logits) {
    EvictWs w;
    const int64_t H = n_heads_of(c);
    int64_t chunks = 0;
    for (int s = 0; s < c->n_seq; ++s) chunks += (int64_t)c->n_layers * c->n_kv_heads * ((c->seq_lens[s] + 4095) / 4096);
    size_t o = 0;
    w.err = o;
    o = align_up(o + sizeof(ErrWord));
    w.ratios = o;
    o = align_up(o + sizeof(double) * (size_t)(n_logits > 0 ? n_logits : 1));
    w.budgets = o;
    o = align_up(o + sizeof(int32_t) * (size_t)H);
    w.budgets_all = o;  // [n_seq][n_logits]: every head's budget when this cache is a head shard
    o = align_up(o + sizeof(int32_t) * (size_t)c->n_seq * (size_t)(n_logits > 0 ? n_logits : 1));
    w.scores = o;
    o = align_up(o + sizeof(float) * (size_t)H * c->max_tokens);
    w.hist = o;
    o = align_up(o + sizeof(uint32_t) * 2048 * (size_t)H);
    w.state = o;
    o = align_up(o + sizeof(HeadSel) * (size_t)H);
    w.chunk_out = o;
    o = align_up(o + sizeof(uint32_t) * (size_t)chunks);
    w.chunk_eqb = o;
    o = align_up(o + sizeof(uint32_t) * (size_t)chunks);
    w.cands = o;
    o = align_up(o + sizeof(uint32_t) * (size_t)H * c->max_tokens);
    w.total = o;
    return w;
}

template <typename T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

lkv_status check_ws(void* ws, size_t have, size_t need) {
    if (!ws) return fail(LKV_ERR_CONTRACT, "workspace is null");
    if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(LKV_ERR_CONTRACT, "workspace must be 256-byte aligned");
    if (have < need) return fail(LKV_ERR_CONTRACT, "workspace too small (" + std::to_string(have) + " < " + std::to_string(need) + ")");
    return LKV_OK;
}

lkv_status check_scorer(const lkv_scorer_desc* s, const lkv_cache_desc* c) {
    if (!s) return fail(LKV_ERR_CONTRACT, "scorer descriptor is null");
    if (c->dtype == LKV_F64) return fail(LKV_ERR_UNSUPPORTED, "fp64 caches are scored by lkv_f64_token_scores");
    if (s->input != LKV_SCORER_K && s->input != LKV_SCORER_KV) return fail(LKV_ERR_CONTRACT, "scorer input must be K or KV");
    if (s->activation != LKV_ACT_SILU && s->activation != LKV_ACT_GELU_ERF) return fail(LKV_ERR_CONTRACT, "unknown activation");
    if (s->hidden < 1 || s->hidden > 256) return fail(LKV_ERR_CONTRACT, "scorer hidden must lie in [1, 256]");
    if (s->n_scorers < 1 || !s->w1t || !s->b1 || !s->w2) return fail(LKV_ERR_CONTRACT, "scorer weights are null");
    const int64_t lo = std::min<int64_t>(0, (int64_t)(c->n_layers - 1) * s->stride_layer) +
                       std::min<int64_t>(0, (int64_t)(c->n_kv_heads - 1) * s->stride_head);
    const int64_t hi = std::max<int64_t>(0, (int64_t)(c->n_layers - 1) * s->stride_layer) +
                       std::max<int64_t>(0, (int64_t)(c->n_kv_heads - 1) * s->stride_head);
    if (lo < 0 || hi >= s->n_scorers) return fail(LKV_ERR_CONTRACT, "scorer index of some (layer, head) out of range");
    return LKV_OK;
}

lkv_status check_ragged(const lkv_ragged_desc* r, int64_t n_heads, int head_dim, int dtype, bool need_rows) {
    if (!r) return fail(LKV_ERR_CONTRACT, "ragged descriptor is null");
    if (r->n_heads != n_heads) return fail(LKV_ERR_CONTRACT, "ragged n_heads mismatch");
    if (r->head_dim != head_dim || r->dtype != dtype) return fail(LKV_ERR_CONTRACT, "ragged head_dim/dtype mismatch");
    if (!r->offsets || !r->lens || !r->positions) return fail(LKV_ERR_CONTRACT, "ragged offsets/lens/positions are null");
    if (need_rows && (!r->keys || !r->values)) return fail(LKV_ERR_CONTRACT, "ragged keys/values are null");
    if (r->decode_slack < 0) return fail(LKV_ERR_CONTRACT, "decode_slack must be >= 0");
    return LKV_OK;
}

// ---- internal launchers shared by lkv_score / lkv_evict ---------------------------------------------
lkv_status run_score(const lkv_cache_desc* c, const lkv_scorer_desc* s, float* scores, cudaStream_t stream,
                     int sms_reserved = 0, uint32_t* hist = nullptr, ErrWord* err = nullptr,
                     bool* hist_made = nullptr, bool clear_hist = true, bool pdl = false) {
    if (hist_made) *hist_made = false;
    ScoreParams p;
    memset(&p, 0, sizeof p);
    p.seq = make_seq(c);
    p.in_mode = s->input;
    p.act = s->activation;
    p.hidden = s->hidden;
    p.stride_layer = s->stride_layer;
    p.stride_head = s->stride_head;
    p.keys = c->keys;
    p.values = c->values;
    p.w1t = s->w1t;
    p.b1 = s->b1;
    p.w2 = s->w2;
    p.scores = scores;
    p.pdl = pdl ? 1 : 0;
    if (score_tc_supported(c->dtype, c->head_dim, s->hidden, s->input)) {
        CUtensorMap mk, mv, mw;
        const uint64_t rows = (uint64_t)n_heads_of(c) * c->max_tokens;
        lkv_status st = make_map_bf16(&mk, c->keys, c->head_dim, rows, 128);
        if (st) return st;
        st = make_map_bf16(&mv, c->values, c->head_dim, rows, 128);
        if (st) return st;
        st = make_map_bf16(&mw, s->w1t, (uint64_t)s->input * c->head_dim, (uint64_t)s->n_scorers * s->hidden,
                           (uint32_t)s->hidden);
        if (st) return st;
        if (hist) {
            if (clear_hist)
                LKV_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2048 * (size_t)n_heads_of(c), stream), "hist clear");
            p.hist = hist;
            p.err = err;
            if (hist_made) *hist_made = true;
        }
        LKV_CUDA(launch_score_tc(p, mk, mv, mw, num_sms() - sms_reserved, stream), "score (tcgen05)");
    } else {
        const int in = s->input * c->head_dim;
        if (score_simt_smem_bytes(in, s->hidden) > 200 * 1024)
            return fail(LKV_ERR_UNSUPPORTED, "scorer too large for the SIMT kernel");
        LKV_CUDA(launch_score_simt(p, c->dtype, num_sms(), stream), "score (simt)");
    }
    return LKV_OK;
}

// `c` may describe a contiguous sub-range of the flat heads of the cache the workspace was laid
// out for: h0 = its first flat head, chunk0 = its first 4096-row select chunk.  Every per-head
// buffer is offset by h0; the ragged rows are addressed through the (absolute) offsets.
lkv_status run_select(const lkv_cache_desc* c, const float* scores, const int32_t* budgets,
                      const lkv_ragged_desc* out, void* ws, const EvictWs& w, bool gather, cudaStream_t stream,
                      bool hist_ready = false, int64_t h0 = 0, int64_t chunk0 = 0) {
    for (int s = 0; s < c->n_seq; ++s)
        if (c->seq_lens[s] > 4096 * 1024) return fail(LKV_ERR_UNSUPPORTED, "top-k supports t <= 4M rows per head");
    SelectParams p;
    memset(&p, 0, sizeof p);
    p.seq = make_seq(c);
    p.scores = scores;
    p.budgets = budgets + h0;
    p.hist = at<uint32_t>(ws, w.hist) + h0 * 2048;
    p.state = at<HeadSel>(ws, w.state) + h0;
    p.chunk_out = at<uint32_t>(ws, w.chunk_out) + chunk0;
    p.chunk_eqb = at<uint32_t>(ws, w.chunk_eqb) + chunk0;
    p.cands = at<uint32_t>(ws, w.cands) + h0 * c->max_tokens;
    p.offsets = out->offsets + h0;
    p.out_pos = out->positions;
    p.out_lens = out->lens + h0;
    p.keys = c->keys;
    p.values = c->values;
    p.out_keys = out->keys;
    p.out_values = out->values;
    p.row_bytes = c->head_dim * elem_bytes(c->dtype);
    p.gather = gather ? 1 : 0;
    p.hist_ready = hist_ready ? 1 : 0;
    p.err = at<ErrWord>(ws, w.err);
    LKV_CUDA(launch_select(p, (int)n_heads_of(c), stream), "select");
    return LKV_OK;
}

// ---- decode workspace -------------------------------------------------------------------------------
struct DecodeWs {
    size_t err, n_items, ch, layer_begin, item_base, new_len, items, part_m, part_l, part_o, total;
    int64_t max_items;
};
DecodeWs decode_layout(const lkv_ragged_desc* r, int G) {
    DecodeWs w;
    w.max_items = r->capacity_rows / kDecMinCh + r->n_heads;
    size_t o = 0;
    w.err = o;
    o = align_up(o + sizeof(ErrWord));
    w.n_items = o;
    o = align_up(o + sizeof(int32_t));
    w.ch = o;  // rows per work item, chosen by the plan
    o = align_up(o + sizeof(int32_t));
    w.layer_begin = o;  // [n_layers + 1] of the plan (n_layers <= n_heads)
    o = align_up(o + sizeof(int32_t) * ((size_t)r->n_heads + 1));
    w.item_base = o;
    o = align_up(o + sizeof(int32_t) * (size_t)r->n_heads);
    w.new_len = o;
    o = align_up(o + sizeof(int32_t) * (size_t)r->n_heads);
    w.items = o;
    o = align_up(o + sizeof(DecodeItem) * (size_t)w.max_items);
    w.part_m = o;
    o = align_up(o + sizeof(float) * (size_t)w.max_items * G);
    w.part_l = o;
    o = align_up(o + sizeof(float) * (size_t)w.max_items * G);
    w.part_o = o;
    o = align_up(o + sizeof(float) * (size_t)w.max_items * G * r->head_dim);
    w.total = o;
    return w;
}

}  // namespace

// =====================================================================================================
extern "C" {

int lkv_abi_version(void) { return LKV_ABI_VERSION; }

uint64_t lkv_launch_count(void) { return lkv_dev::launch_count(); }

const char* lkv_last_error(void) { return g_err.c_str(); }

const char* lkv_status_name(int s) {
    switch (s) {
        case LKV_OK: return "ok";
        case LKV_ERR_CONTRACT: return "contract_error";
        case LKV_ERR_NUMERIC: return "numeric_error";
        case LKV_ERR_BUDGET: return "budget_error";
        case LKV_ERR_OVERFLOW_GUARD: return "overflow_guard_error";
        case LKV_ERR_DEGENERATE_MASK: return "degenerate_mask_error";
        case LKV_ERR_CUDA: return "cuda_error";
        case LKV_ERR_UNSUPPORTED: return "unsupported";
        case LKV_ERR_NCCL: return "nccl_error";
    }
    return "unknown";
}

lkv_status lkv_device_check(void) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(LKV_ERR_UNSUPPORTED, "this library is built for sm_100a (B200); found sm_" + std::to_string(major) +
                                             std::to_string(minor));
    return LKV_OK;
}

size_t lkv_workspace_bytes(const lkv_cache_desc* cache, int32_t n_logits) {
    if (check_cache(cache, false)) return 0;
    return evict_layout(cache, n_logits).total;
}

lkv_status lkv_workspace_init(void* ws, size_t bytes, lkv_stream_t stream) {
    if (!ws || bytes < sizeof(ErrWord)) return fail(LKV_ERR_CONTRACT, "workspace is null or too small");
    LKV_CUDA(cudaMemsetAsync(ws, 0, sizeof(ErrWord), (cudaStream_t)stream), "workspace init");
    return LKV_OK;
}

lkv_status lkv_workspace_status(void* ws, lkv_stream_t stream) {
    if (!ws) return fail(LKV_ERR_CONTRACT, "workspace is null");
    ErrWord h{0, 0};
    LKV_CUDA(cudaMemcpyAsync(&h, ws, sizeof h, cudaMemcpyDeviceToHost, (cudaStream_t)stream), "status read");
    LKV_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
    if (h.code != 0) {
        LKV_CUDA(cudaMemsetAsync(ws, 0, sizeof(ErrWord), (cudaStream_t)stream), "status clear");
        LKV_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
        return fail((lkv_status)h.code, std::string("device-side ") + lkv_status_name(h.code) + " (detail " +
                                            std::to_string(h.detail) + ")");
    }
    return LKV_OK;
}

int64_t lkv_ragged_capacity(const lkv_cache_desc* c, double R, int32_t slack) {
    if (check_cache(c, false)) return -1;
    const int64_t n = (int64_t)c->n_layers * c->n_kv_heads;
    int64_t rows = 0;
    for (int s = 0; s < c->n_seq; ++s) rows += llround(R * n * c->seq_lens[s]) + n;  // +n: FLOOR-mode margin
    return rows + n_heads_of(c) * (int64_t)slack;
}

int64_t lkv_ragged_capacity_shard(const lkv_cache_desc* c, int32_t n_logits, double R, int32_t slack) {
    if (check_cache(c, false) || n_logits < 1) return -1;
    const int64_t nl = (int64_t)c->n_layers * c->n_kv_heads;
    int64_t rows = 0;
    for (int s = 0; s < c->n_seq; ++s)  // the shard holds at most the whole budget, at most every row
        rows += std::min<int64_t>(llround(R * n_logits * c->seq_lens[s]) + n_logits, nl * c->seq_lens[s]);
    return rows + n_heads_of(c) * (int64_t)slack;
}

lkv_status lkv_budgets(const double* logits, int32_t n, double R, int32_t mode, const int32_t* seq_lens, int32_t n_seq,
                       int32_t slack, double* ratios, int32_t* budgets, int64_t* offsets, void* ws, size_t ws_bytes,
                       lkv_stream_t stream) {
    if (!(R > 0.0 && R < 1.0)) return fail(LKV_ERR_BUDGET, "target ratio must lie in (0,1)");  // policy.cpp:111
    if (n < 1 || n > 3072) return fail(LKV_ERR_CONTRACT, "allocate_budgets: need 1 <= n <= 3072 head logits");
    if (mode != LKV_BUDGET_FLOOR && mode != LKV_BUDGET_EXACT) return fail(LKV_ERR_CONTRACT, "unknown budget mode");
    if (n_seq < 1 || n_seq > LKV_MAX_SEQ || !seq_lens) return fail(LKV_ERR_CONTRACT, "bad sequence table");
    for (int s = 0; s < n_seq; ++s)
        if (seq_lens[s] < 1) return fail(LKV_ERR_CONTRACT, "freeze_budgets: t must be >= 1");  // policy.cpp:123
    if (!logits || !budgets) return fail(LKV_ERR_CONTRACT, "logits/budgets are null");
    if (slack < 0) return fail(LKV_ERR_CONTRACT, "decode_slack must be >= 0");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    BudgetParams p;
    memset(&p, 0, sizeof p);
    p.logits = logits;
    p.n = n;
    p.mode = mode;
    p.R = R;
    p.n_seq = n_seq;
    p.slack = slack;
    p.ratios_out = ratios;
    p.budgets_out = budgets;
    p.offsets_out = offsets;
    p.err = at<ErrWord>(ws, 0);
    for (int s = 0; s < n_seq; ++s) p.seq_len[s] = seq_lens[s];
    LKV_CUDA(launch_budgets(p, (cudaStream_t)stream), "budgets");
    return LKV_OK;
}

static lkv_status budgets_shard_impl(const double* logits, int32_t n, double R, int32_t mode, const int32_t* seq_lens,
                                     int32_t n_seq, int32_t slack, int32_t head_begin, const int32_t* head_ids,
                                     int32_t n_local, double* ratios, int32_t* budgets_all, int32_t* budgets_local,
                                     int64_t* offsets_local, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (head_ids) {
        if (n_local < 1 || n_local > n) return fail(LKV_ERR_CONTRACT, "budgets_heads: need 1 <= n_local <= n");
    } else if (n_local < 1 || head_begin < 0 || (int64_t)head_begin + n_local > n) {
        return fail(LKV_ERR_CONTRACT, "budgets_shard: need 0 <= head_begin and head_begin + n_local <= n");
    }
    if (!budgets_all || !budgets_local) return fail(LKV_ERR_CONTRACT, "budgets_shard: null budget buffers");
    if (!(R > 0.0 && R < 1.0)) return fail(LKV_ERR_BUDGET, "target ratio must lie in (0,1)");  // policy.cpp:111
    if (n > 3072) return fail(LKV_ERR_CONTRACT, "allocate_budgets: need 1 <= n <= 3072 head logits");
    if (mode != LKV_BUDGET_FLOOR && mode != LKV_BUDGET_EXACT) return fail(LKV_ERR_CONTRACT, "unknown budget mode");
    if (n_seq < 1 || n_seq > LKV_MAX_SEQ || !seq_lens) return fail(LKV_ERR_CONTRACT, "bad sequence table");
    for (int s = 0; s < n_seq; ++s)
        if (seq_lens[s] < 1) return fail(LKV_ERR_CONTRACT, "freeze_budgets: t must be >= 1");  // policy.cpp:123
    if (!logits) return fail(LKV_ERR_CONTRACT, "logits are null");
    if (slack < 0) return fail(LKV_ERR_CONTRACT, "decode_slack must be >= 0");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    BudgetParams p;
    memset(&p, 0, sizeof p);
    p.logits = logits;
    p.n = n;
    p.mode = mode;
    p.R = R;
    p.n_seq = n_seq;
    p.slack = slack;
    p.ratios_out = ratios;
    p.budgets_out = budgets_all;
    p.offsets_out = offsets_local;
    p.local_begin = head_ids ? 0 : head_begin;
    p.local_count = n_local;
    p.local_ids = head_ids;
    p.budgets_local_out = budgets_local;
    p.err = at<ErrWord>(ws, 0);
    for (int s = 0; s < n_seq; ++s) p.seq_len[s] = seq_lens[s];
    LKV_CUDA(launch_budgets(p, (cudaStream_t)stream), "budgets (shard)");
    return LKV_OK;
}

lkv_status lkv_budgets_shard(const double* logits, int32_t n, double R, int32_t mode, const int32_t* seq_lens,
                             int32_t n_seq, int32_t slack, int32_t head_begin, int32_t n_local, double* ratios,
                             int32_t* budgets_all, int32_t* budgets_local, int64_t* offsets_local, void* ws,
                             size_t ws_bytes, lkv_stream_t stream) {
    return budgets_shard_impl(logits, n, R, mode, seq_lens, n_seq, slack, head_begin, nullptr, n_local, ratios,
                              budgets_all, budgets_local, offsets_local, ws, ws_bytes, stream);
}

lkv_status lkv_budgets_heads(const double* logits, int32_t n, double R, int32_t mode, const int32_t* seq_lens,
                             int32_t n_seq, int32_t slack, const int32_t* head_ids, int32_t n_local, double* ratios,
                             int32_t* budgets_all, int32_t* budgets_local, int64_t* offsets_local, void* ws,
                             size_t ws_bytes, lkv_stream_t stream) {
    if (!head_ids) return fail(LKV_ERR_CONTRACT, "budgets_heads: head_ids are null");
    return budgets_shard_impl(logits, n, R, mode, seq_lens, n_seq, slack, 0, head_ids, n_local, ratios, budgets_all,
                              budgets_local, offsets_local, ws, ws_bytes, stream);
}

lkv_status lkv_freeze_budgets(const double* ratios, int32_t n, double R, int32_t mode, const int32_t* seq_lens,
                              int32_t n_seq, int32_t slack, int32_t* budgets, int64_t* offsets, void* ws,
                              size_t ws_bytes, lkv_stream_t stream) {
    if (mode != LKV_BUDGET_FLOOR && mode != LKV_BUDGET_EXACT) return fail(LKV_ERR_CONTRACT, "unknown budget mode");
    if (mode == LKV_BUDGET_EXACT && !(R > 0.0 && R < 1.0)) return fail(LKV_ERR_BUDGET, "target ratio must lie in (0,1)");
    if (n < 1 || n > 3072) return fail(LKV_ERR_CONTRACT, "freeze_budgets: need 1 <= n <= 3072 ratios");
    if (n_seq < 1 || n_seq > LKV_MAX_SEQ || !seq_lens) return fail(LKV_ERR_CONTRACT, "bad sequence table");
    for (int s = 0; s < n_seq; ++s)
        if (seq_lens[s] < 1) return fail(LKV_ERR_CONTRACT, "freeze_budgets: t must be >= 1");  // policy.cpp:123
    if (!ratios || !budgets) return fail(LKV_ERR_CONTRACT, "ratios/budgets are null");
    if (slack < 0) return fail(LKV_ERR_CONTRACT, "decode_slack must be >= 0");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    BudgetParams p;
    memset(&p, 0, sizeof p);
    p.ratios_in = ratios;
    p.n = n;
    p.mode = mode;
    p.R = R;
    p.n_seq = n_seq;
    p.slack = slack;
    p.budgets_out = budgets;
    p.offsets_out = offsets;
    p.err = at<ErrWord>(ws, 0);
    for (int s = 0; s < n_seq; ++s) p.seq_len[s] = seq_lens[s];
    LKV_CUDA(launch_budgets(p, (cudaStream_t)stream), "freeze budgets");
    return LKV_OK;
}

lkv_status lkv_ragged_offsets(const int32_t* budgets, int32_t n_heads, int32_t slack, int64_t* offsets,
                              lkv_stream_t stream) {
    if (!budgets || !offsets || n_heads < 1 || slack < 0) return fail(LKV_ERR_CONTRACT, "bad ragged_offsets arguments");
    LKV_CUDA(launch_offsets(budgets, n_heads, slack, offsets, (cudaStream_t)stream), "offsets");
    return LKV_OK;
}

lkv_status lkv_score(const lkv_cache_desc* c, const lkv_scorer_desc* s, float* scores, void* ws, size_t ws_bytes,
                     lkv_stream_t stream) {
    lkv_status st = check_cache(c, true);
    if (st) return st;
    if ((st = check_scorer(s, c))) return st;
    if (!scores) return fail(LKV_ERR_CONTRACT, "scores is null");
    (void)ws;
    (void)ws_bytes;
    return run_score(c, s, scores, (cudaStream_t)stream);
}

lkv_status lkv_select(const lkv_cache_desc* c, const float* scores, const int32_t* budgets, const lkv_ragged_desc* out,
                      int32_t gather, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    lkv_status st = check_cache(c, gather != 0);
    if (st) return st;
    if (c->dtype == LKV_F64) return fail(LKV_ERR_UNSUPPORTED, "fp64 scores are selected by lkv_f64_select");
    if ((st = check_ragged(out, n_heads_of(c), c->head_dim, c->dtype, gather != 0))) return st;
    if (!scores || !budgets) return fail(LKV_ERR_CONTRACT, "scores/budgets are null");
    const EvictWs w = evict_layout(c, 1);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    return run_select(c, scores, budgets, out, ws, w, gather != 0, (cudaStream_t)stream);
}

lkv_status lkv_compact(const lkv_cache_desc* c, const lkv_ragged_desc* out, void* ws, size_t ws_bytes,
                       lkv_stream_t stream) {
    lkv_status st = check_cache(c, true);
    if (st) return st;
    if ((st = check_ragged(out, n_heads_of(c), c->head_dim, c->dtype, true))) return st;
    if ((st = check_ws(ws, ws_bytes, sizeof(ErrWord)))) return st;
    CompactParams p;
    memset(&p, 0, sizeof p);
    p.seq = make_seq(c);
    p.offsets = out->offsets;
    p.lens = out->lens;
    p.positions = out->positions;
    p.keys = c->keys;
    p.values = c->values;
    p.out_keys = out->keys;
    p.out_values = out->values;
    p.row_bytes = c->head_dim * elem_bytes(c->dtype);
    p.err = at<ErrWord>(ws, 0);  // out-of-range positions / overrun heads -> contract_error
    LKV_CUDA(launch_compact(p, (int)n_heads_of(c), (cudaStream_t)stream), "compact");
    return LKV_OK;
}

static lkv_status trace_params(const lkv_cache_desc* c, const int32_t* masks, int64_t mask_ld, void* ws,
                               size_t ws_bytes, TraceParams* p) {
    lkv_status st = check_cache(c, false);
    if (st) return st;
    if (!masks) return fail(LKV_ERR_CONTRACT, "cache_from_trace: masks are null");
    int64_t tmax = 0;
    for (int s = 0; s < c->n_seq; ++s) tmax = std::max<int64_t>(tmax, c->seq_lens[s]);
    if (mask_ld < tmax) return fail(LKV_ERR_CONTRACT, "cache_from_trace: mask length mismatch");  // model.cpp:300
    for (int s = 0; s < c->n_seq; ++s)
        if (c->seq_lens[s] > 4096 * 1024) return fail(LKV_ERR_UNSUPPORTED, "cache_from_trace supports t <= 4M rows");
    const EvictWs w = evict_layout(c, 1);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    memset(p, 0, sizeof *p);
    p->seq = make_seq(c);
    p->masks = masks;
    p->mask_ld = mask_ld;
    p->chunk_cnt = at<uint32_t>(ws, w.chunk_out);
    p->err = at<ErrWord>(ws, w.err);
    p->row_bytes = c->head_dim * elem_bytes(c->dtype);
    return LKV_OK;
}

lkv_status lkv_mask_counts(const lkv_cache_desc* c, const int32_t* masks, int64_t mask_ld, int32_t* counts, void* ws,
                           size_t ws_bytes, lkv_stream_t stream) {
    TraceParams p;
    lkv_status st = trace_params(c, masks, mask_ld, ws, ws_bytes, &p);
    if (st) return st;
    if (!counts) return fail(LKV_ERR_CONTRACT, "mask_counts: counts is null");
    p.counts = counts;
    LKV_CUDA(launch_trace_counts(p, (int)n_heads_of(c), (cudaStream_t)stream), "mask counts");
    return LKV_OK;
}

lkv_status lkv_cache_from_trace(const lkv_cache_desc* c, const int32_t* masks, int64_t mask_ld,
                                const lkv_ragged_desc* out, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    TraceParams p;
    lkv_status st = trace_params(c, masks, mask_ld, ws, ws_bytes, &p);
    if (st) return st;
    if ((st = check_cache(c, true))) return st;
    if ((st = check_ragged(out, n_heads_of(c), c->head_dim, c->dtype, true))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    p.counts = out->lens;
    p.offsets = out->offsets;
    p.capacity = out->capacity_rows;
    p.out_pos = out->positions;
    p.keys = c->keys;
    p.values = c->values;
    p.out_keys = out->keys;
    p.out_values = out->values;
    p.gather = 1;
    LKV_CUDA(launch_trace_counts(p, (int)n_heads_of(c), s), "mask counts");
    LKV_CUDA(launch_offsets(out->lens, (int)n_heads_of(c), out->decode_slack, out->offsets, s), "offsets");
    LKV_CUDA(launch_trace_emit(p, s), "cache_from_trace emit");
    return LKV_OK;
}

// score -> budget -> top-k -> compact on ONE stream as one programmatic-dependent-launch chain:
//   K2 budgets (1 CTA, triggers its dependents at once) -> K1 scorer (PDL: runs on the other SMs
//   while K2 solves; every K1 CTA waits for K2 before it completes) -> K3 plan -> K3+K4 emit (each
//   waits for its predecessor).  No side stream, no flag: K2 is resident before K1 launches, so
//   every wait makes progress on any SM partitioning, and the chain is graph-capturable.
static lkv_status evict_impl(const lkv_cache_desc* c, const lkv_scorer_desc* s, const double* logits, int n,
                             int head_begin, bool shard, const int32_t* head_ids, double R, int32_t mode,
                             const lkv_ragged_desc* out,
                             float* scores_out, double* ratios_out, int32_t* budgets_out, void* ws, size_t ws_bytes,
                             cudaStream_t strm) {
    lkv_status st = check_cache(c, true);
    if (st) return st;
    if ((st = check_scorer(s, c))) return st;
    if ((st = check_ragged(out, n_heads_of(c), c->head_dim, c->dtype, true))) return st;
    const EvictWs w = evict_layout(c, n);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    int32_t* budgets = budgets_out ? budgets_out : at<int32_t>(ws, w.budgets);
    double* ratios = ratios_out ? ratios_out : at<double>(ws, w.ratios);
    float* scores = scores_out ? scores_out : at<float>(ws, w.scores);
    // the tcgen05 scorer fuses top-k pass 1 (the histogram) into its epilogue: clear it before
    // K2 (a memset between K2 and K1 would break the launch chain)
    const bool tc = score_tc_supported(c->dtype, c->head_dim, s->hidden, s->input);
    uint32_t* hist = at<uint32_t>(ws, w.hist);
    if (tc) LKV_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2048 * (size_t)n_heads_of(c), strm), "hist clear");
    if (shard)
        st = budgets_shard_impl(logits, n, R, mode, c->seq_lens, c->n_seq, out->decode_slack, head_begin, head_ids,
                                c->n_layers * c->n_kv_heads, ratios, at<int32_t>(ws, w.budgets_all), budgets,
                                out->offsets, ws, ws_bytes, (lkv_stream_t)strm);
    else
        st = lkv_budgets(logits, n, R, mode, c->seq_lens, c->n_seq, out->decode_slack, ratios, budgets, out->offsets,
                         ws, ws_bytes, (lkv_stream_t)strm);
    if (st) return st;
    // K1 leaves one SM to K2.  The SIMT scorer (fp32 inputs) is launched normally: it runs after K2
    // and the histogram kernel of the select reads the budgets.
    bool hist_made = false;
    if ((st = run_score(c, s, scores, strm, /*sms_reserved=*/tc ? 1 : 0, hist, at<ErrWord>(ws, w.err), &hist_made,
                        /*clear_hist=*/false, /*pdl=*/tc)))
        return st;
    return run_select(c, scores, budgets, out, ws, w, true, strm, hist_made);
}

lkv_status lkv_evict(const lkv_cache_desc* c, const lkv_scorer_desc* s, const double* logits, double R, int32_t mode,
                     const lkv_ragged_desc* out, float* scores_out, double* ratios_out, int32_t* budgets_out, void* ws,
                     size_t ws_bytes, lkv_stream_t stream) {
    if (!c) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    return evict_impl(c, s, logits, c->n_layers * c->n_kv_heads, 0, false, nullptr, R, mode, out, scores_out, ratios_out,
                      budgets_out, ws, ws_bytes, (cudaStream_t)stream);
}

lkv_status lkv_evict_budgets(const lkv_cache_desc* c, const lkv_scorer_desc* s, const int32_t* budgets,
                             const lkv_ragged_desc* out, float* scores_out, void* ws, size_t ws_bytes,
                             lkv_stream_t stream) {
    lkv_status st = check_cache(c, true);
    if (st) return st;
    if ((st = check_scorer(s, c))) return st;
    if ((st = check_ragged(out, n_heads_of(c), c->head_dim, c->dtype, true))) return st;
    if (!budgets) return fail(LKV_ERR_CONTRACT, "budgets are null");
    const EvictWs w = evict_layout(c, 1);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    cudaStream_t strm = (cudaStream_t)stream;
    float* scores = scores_out ? scores_out : at<float>(ws, w.scores);
    bool hist_made = false;  // K1 fuses top-k pass 1 into its epilogue (tcgen05 path)
    if ((st = run_score(c, s, scores, strm, 0, at<uint32_t>(ws, w.hist), at<ErrWord>(ws, w.err), &hist_made))) return st;
    return run_select(c, scores, budgets, out, ws, w, true, strm, hist_made);
}

lkv_status lkv_evict_shard(const lkv_cache_desc* c, const lkv_scorer_desc* s, const double* logits, int32_t n_logits,
                           int32_t head_begin, double R, int32_t mode, const lkv_ragged_desc* out, float* scores_out,
                           double* ratios_out, int32_t* budgets_out, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!c) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    if (n_logits < 1 || head_begin < 0 || (int64_t)head_begin + (int64_t)c->n_layers * c->n_kv_heads > n_logits)
        return fail(LKV_ERR_CONTRACT, "evict_shard: the shard's heads must lie inside the n_logits global heads");
    return evict_impl(c, s, logits, n_logits, head_begin, true, nullptr, R, mode, out, scores_out, ratios_out,
                      budgets_out, ws, ws_bytes, (cudaStream_t)stream);
}

lkv_status lkv_evict_heads(const lkv_cache_desc* c, const lkv_scorer_desc* s, const double* logits, int32_t n_logits,
                           const int32_t* head_ids, double R, int32_t mode, const lkv_ragged_desc* out,
                           float* scores_out, double* ratios_out, int32_t* budgets_out, void* ws, size_t ws_bytes,
                           lkv_stream_t stream) {
    if (!c) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    if (!head_ids) return fail(LKV_ERR_CONTRACT, "evict_heads: head_ids are null");
    if (n_logits < 1 || (int64_t)c->n_layers * c->n_kv_heads > n_logits)
        return fail(LKV_ERR_CONTRACT, "evict_heads: more local heads than global heads");
    return evict_impl(c, s, logits, n_logits, 0, true, head_ids, R, mode, out, scores_out, ratios_out, budgets_out, ws,
                      ws_bytes, (cudaStream_t)stream);
}

// Eviction of a host-resident (pinned, device-mapped) dense cache, pipelined per chunk =
// (sequence, layer group) over three streams:
//   copy stream : K (and V for [k;v] scorers) of chunk i uploaded H2D;
//   main stream : chunk i scored (K1 + fused histogram) and selected/gathered (K3+K4) as soon as
//                 its K landed; its kept V rows are read straight from the mapped host V (only
//                 rho of V crosses PCIe);
//   d2h stream  : chunk i's compacted rows copied back to the pinned host cache while later
//                 chunks are still uploading (PCIe is full duplex).
// The D2H ranges need the ragged offsets on the host: K2 runs first on the side stream and
// its offsets are read back once (all K uploads are already queued, so the wait is hidden).
static lkv_status evict_host_impl(const lkv_cache_desc* hc, void* dev_keys, void* dev_values, const lkv_scorer_desc* s,
                                  const double* logits, int32_t n_logits, int32_t head_begin, bool shard,
                                  const int32_t* head_ids, double R,
                                  int32_t mode, const lkv_ragged_desc* out, const lkv_ragged_desc* host_out,
                                  int32_t layers_per_chunk, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    lkv_status st = check_cache(hc, true);
    if (st) return st;
    if ((st = check_scorer(s, hc))) return st;
    if ((st = check_ragged(out, n_heads_of(hc), hc->head_dim, hc->dtype, true))) return st;
    if (!dev_keys) return fail(LKV_ERR_CONTRACT, "dev_keys (device staging for K) is null");
    const bool kv = s->input == LKV_SCORER_KV;
    if (kv && !dev_values) return fail(LKV_ERR_CONTRACT, "[k;v] scorers need dev_values staging");
    if (layers_per_chunk < 1) layers_per_chunk = 1;
    if (host_out && (!host_out->keys || !host_out->values || !host_out->positions || !host_out->offsets ||
                     !host_out->lens || host_out->capacity_rows < out->capacity_rows))
        return fail(LKV_ERR_CONTRACT, "host_out buffers missing or too small");
    // host V must be device-accessible (pinned + mapped): use its device alias for the gather
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, hc->values) != cudaSuccess || pa.type != cudaMemoryTypeHost || !pa.devicePointer)
        return fail(LKV_ERR_CONTRACT, "host values must be pinned, device-mapped memory (cudaHostAlloc)");
    if (host_out) {
        cudaPointerAttributes po{};
        if (cudaPointerGetAttributes(&po, host_out->offsets) != cudaSuccess || po.type != cudaMemoryTypeHost)
            return fail(LKV_ERR_CONTRACT, "host_out buffers must be pinned host memory");
    }
    const char* v_dev_alias = static_cast<const char*>(pa.devicePointer);
    const int n = n_logits;
    const EvictWs w = evict_layout(hc, n);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    cudaStream_t strm = (cudaStream_t)stream;
    cudaStream_t side = side_stream(), cs = copy_stream(), ds = d2h_stream();
    if (!side || !cs || !ds) return fail(LKV_ERR_CUDA, "helper stream creation failed");
    const size_t esz = elem_bytes(hc->dtype);
    const size_t rowb = (size_t)hc->head_dim * esz;
    const size_t head_bytes = (size_t)hc->max_tokens * rowb;
    const int H = hc->n_kv_heads, L = hc->n_layers;
    int32_t* budgets = at<int32_t>(ws, w.budgets);
    float* scores = at<float>(ws, w.scores);
    uint32_t* hist = at<uint32_t>(ws, w.hist);

    std::vector<cudaEvent_t> evs;
    struct Evs {
        std::vector<cudaEvent_t>& v;
        ~Evs() {
            for (auto e : v) cudaEventDestroy(e);
        }
    } guard{evs};
    auto mk = [&]() -> cudaEvent_t {
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) evs.push_back(e);
        return e;
    };
    cudaEvent_t start = mk(), join = mk();
    if (!start || !join) return fail(LKV_ERR_CUDA, "event creation failed");
    LKV_CUDA(cudaEventRecord(start, strm), "event record");
    LKV_CUDA(cudaStreamWaitEvent(side, start, 0), "stream wait");
    LKV_CUDA(cudaStreamWaitEvent(cs, start, 0), "stream wait");
    LKV_CUDA(cudaStreamWaitEvent(ds, start, 0), "stream wait");
    // K2 on the side stream; its offsets go to the host when the compacted cache is copied back
    if (shard)
        st = budgets_shard_impl(logits, n, R, mode, hc->seq_lens, hc->n_seq, out->decode_slack, head_begin, head_ids,
                                hc->n_layers * hc->n_kv_heads, at<double>(ws, w.ratios), at<int32_t>(ws, w.budgets_all),
                                budgets, out->offsets, ws, ws_bytes, (lkv_stream_t)side);
    else
        st = lkv_budgets(logits, n, R, mode, hc->seq_lens, hc->n_seq, out->decode_slack, at<double>(ws, w.ratios),
                         budgets, out->offsets, ws, ws_bytes, (lkv_stream_t)side);
    if (st) return st;
    const int64_t n_heads = n_heads_of(hc);
    if (host_out)
        LKV_CUDA(cudaMemcpyAsync(host_out->offsets, out->offsets, sizeof(int64_t) * (n_heads + 1), cudaMemcpyDeviceToHost,
                                 side),
                 "offsets D2H");
    LKV_CUDA(cudaEventRecord(join, side), "event record");
    // 1. queue every chunk's upload on the copy stream
    struct Chunk {
        int sq, l0, nl;
        int64_t h0, c0;
        cudaEvent_t ready;
    };
    std::vector<Chunk> chunks;
    int64_t cbase = 0;
    for (int sq = 0; sq < hc->n_seq; ++sq) {
        const int64_t cph = (hc->seq_lens[sq] + 4095) / 4096;  // select chunks per head
        for (int l0 = 0; l0 < L; l0 += layers_per_chunk) {
            Chunk ch;
            ch.sq = sq;
            ch.l0 = l0;
            ch.nl = std::min(layers_per_chunk, L - l0);
            ch.h0 = (int64_t)(sq * L + l0) * H;
            ch.c0 = cbase + (int64_t)l0 * H * cph;
            const size_t bytes = (size_t)ch.nl * H * head_bytes;
            LKV_CUDA(cudaMemcpyAsync(static_cast<char*>(dev_keys) + ch.h0 * head_bytes,
                                     static_cast<const char*>(hc->keys) + ch.h0 * head_bytes, bytes,
                                     cudaMemcpyHostToDevice, cs),
                     "K upload");
            if (kv)
                LKV_CUDA(cudaMemcpyAsync(static_cast<char*>(dev_values) + ch.h0 * head_bytes,
                                         static_cast<const char*>(hc->values) + ch.h0 * head_bytes, bytes,
                                         cudaMemcpyHostToDevice, cs),
                         "V upload");
            if (!(ch.ready = mk())) return fail(LKV_ERR_CUDA, "event creation failed");
            LKV_CUDA(cudaEventRecord(ch.ready, cs), "event record");
            chunks.push_back(ch);
        }
        cbase += (int64_t)L * H * cph;
    }
    // 2. the host needs the ragged offsets to size the per-chunk copy-back
    if (host_out) LKV_CUDA(cudaEventSynchronize(join), "offsets wait");
    LKV_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2048 * (size_t)n_heads, strm), "hist clear");
    LKV_CUDA(cudaStreamWaitEvent(strm, join, 0), "stream wait");
    // 3. per chunk: score -> select + gather -> copy back
    for (const Chunk& ch : chunks) {
        LKV_CUDA(cudaStreamWaitEvent(strm, ch.ready, 0), "stream wait");
        lkv_cache_desc sub = *hc;
        sub.n_seq = 1;
        sub.n_layers = ch.nl;
        sub.keys = static_cast<char*>(dev_keys) + ch.h0 * head_bytes;
        sub.values = kv ? static_cast<char*>(dev_values) + ch.h0 * head_bytes : sub.keys;
        sub.seq_lens = hc->seq_lens + ch.sq;
        lkv_scorer_desc ss = *s;
        const int64_t sc0 = (int64_t)ch.l0 * s->stride_layer;
        const size_t in = (size_t)s->input * hc->head_dim;
        ss.w1t = static_cast<const char*>(s->w1t) + (size_t)sc0 * s->hidden * in * esz;
        ss.b1 = s->b1 + sc0 * s->hidden;
        ss.w2 = s->w2 + sc0 * s->hidden;
        ss.n_scorers = (int32_t)(s->n_scorers - sc0);
        float* sc = scores + ch.h0 * hc->max_tokens;
        bool made = false;
        if ((st = run_score(&sub, &ss, sc, strm, 0, hist + ch.h0 * 2048, at<ErrWord>(ws, w.err), &made,
                            /*clear_hist=*/false)))
            return st;
        lkv_cache_desc gsrc = sub;
        gsrc.values = kv ? sub.values : v_dev_alias + ch.h0 * head_bytes;
        if ((st = run_select(&gsrc, sc, budgets, out, ws, w, true, strm, made, ch.h0, ch.c0))) return st;
        if (!host_out) continue;
        cudaEvent_t done = mk();
        if (!done) return fail(LKV_ERR_CUDA, "event creation failed");
        LKV_CUDA(cudaEventRecord(done, strm), "event record");
        LKV_CUDA(cudaStreamWaitEvent(ds, done, 0), "stream wait");
        const int64_t nh = (int64_t)ch.nl * H;
        const int64_t r0 = host_out->offsets[ch.h0], r1 = host_out->offsets[ch.h0 + nh];
        if (r0 < 0 || r1 < r0 || r1 > out->capacity_rows)  // K2 failed (latched in the workspace) or capacity short
            return fail(LKV_ERR_CONTRACT, "ragged offsets exceed the output capacity (see lkv_workspace_status)");
        if (r1 > r0) {
            LKV_CUDA(cudaMemcpyAsync(static_cast<char*>(host_out->keys) + r0 * rowb,
                                     static_cast<const char*>(out->keys) + r0 * rowb, (r1 - r0) * rowb,
                                     cudaMemcpyDeviceToHost, ds),
                     "D2H");
            LKV_CUDA(cudaMemcpyAsync(static_cast<char*>(host_out->values) + r0 * rowb,
                                     static_cast<const char*>(out->values) + r0 * rowb, (r1 - r0) * rowb,
                                     cudaMemcpyDeviceToHost, ds),
                     "D2H");
            LKV_CUDA(cudaMemcpyAsync(host_out->positions + r0, out->positions + r0, (r1 - r0) * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, ds),
                     "D2H");
        }
        LKV_CUDA(cudaMemcpyAsync(host_out->lens + ch.h0, out->lens + ch.h0, nh * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, ds),
                 "D2H");
    }
    if (host_out) {
        cudaEvent_t back = mk();
        if (!back) return fail(LKV_ERR_CUDA, "event creation failed");
        LKV_CUDA(cudaEventRecord(back, ds), "event record");
        LKV_CUDA(cudaStreamWaitEvent(strm, back, 0), "stream wait");
    }
    return LKV_OK;
}

lkv_status lkv_evict_host(const lkv_cache_desc* hc, void* dev_keys, void* dev_values, const lkv_scorer_desc* s,
                          const double* logits, double R, int32_t mode, const lkv_ragged_desc* out,
                          const lkv_ragged_desc* host_out, int32_t layers_per_chunk, void* ws, size_t ws_bytes,
                          lkv_stream_t stream) {
    if (!hc) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    return evict_host_impl(hc, dev_keys, dev_values, s, logits, hc->n_layers * hc->n_kv_heads, 0, false, nullptr, R, mode, out,
                           host_out, layers_per_chunk, ws, ws_bytes, stream);
}

lkv_status lkv_evict_host_shard(const lkv_cache_desc* hc, void* dev_keys, void* dev_values, const lkv_scorer_desc* s,
                                const double* logits, int32_t n_logits, int32_t head_begin, double R, int32_t mode,
                                const lkv_ragged_desc* out, const lkv_ragged_desc* host_out, int32_t layers_per_chunk,
                                void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!hc) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    if (n_logits < 1 || head_begin < 0 || (int64_t)head_begin + (int64_t)hc->n_layers * hc->n_kv_heads > n_logits)
        return fail(LKV_ERR_CONTRACT, "evict_host_shard: the shard's heads must lie inside the n_logits global heads");
    return evict_host_impl(hc, dev_keys, dev_values, s, logits, n_logits, head_begin, true, nullptr, R, mode, out,
                           host_out, layers_per_chunk, ws, ws_bytes, stream);
}

lkv_status lkv_evict_host_heads(const lkv_cache_desc* hc, void* dev_keys, void* dev_values, const lkv_scorer_desc* s,
                                const double* logits, int32_t n_logits, const int32_t* head_ids, double R, int32_t mode,
                                const lkv_ragged_desc* out, const lkv_ragged_desc* host_out, int32_t layers_per_chunk,
                                void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!hc) return fail(LKV_ERR_CONTRACT, "cache descriptor is null");
    if (!head_ids) return fail(LKV_ERR_CONTRACT, "evict_host_heads: head_ids are null");
    if (n_logits < 1 || (int64_t)hc->n_layers * hc->n_kv_heads > n_logits)
        return fail(LKV_ERR_CONTRACT, "evict_host_heads: more local heads than global heads");
    return evict_host_impl(hc, dev_keys, dev_values, s, logits, n_logits, 0, true, head_ids, R, mode, out, host_out,
                           layers_per_chunk, ws, ws_bytes, stream);
}

// ---- Soft-TopK (training) -------------------------------------------------
lkv_status lkv_soft_topk_fwd(const double* x, const double* noise, double noise_scale, int32_t n_seg, int32_t n,
                             int64_t ld, const double* k, double tau, double* values, double* density,
                             float* values_f32, double* lambda, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!(tau > 0.0)) return fail(LKV_ERR_CONTRACT, "soft_topk_forward: tau must be positive");  // soft_topk.cpp:112
    if (n < 1) return fail(LKV_ERR_CONTRACT, "soft_topk_forward: empty scores");              // :114
    if (n_seg < 1 || ld < n) return fail(LKV_ERR_CONTRACT, "soft_topk: need n_seg >= 1 and ld >= n");
    if (!x || !k || !values) return fail(LKV_ERR_CONTRACT, "soft_topk: null buffer");
    if (noise && !std::isfinite(noise_scale)) return fail(LKV_ERR_CONTRACT, "soft_topk: noise_scale must be finite");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    SoftTopKParams p;
    memset(&p, 0, sizeof p);
    p.n_seg = n_seg;
    p.n = n;
    p.ld = ld;
    p.tau = tau;
    p.noise_scale = noise_scale;
    p.x = x;
    p.noise = noise;
    p.k = k;
    p.values = values;
    p.density = density;
    p.values_f32 = values_f32;
    p.lambda = lambda;
    p.err = at<ErrWord>(ws, 0);
    LKV_CUDA(launch_soft_topk_fwd(p, (cudaStream_t)stream), "soft topk forward");
    return LKV_OK;
}

lkv_status lkv_soft_topk_vjp(const double* density, const double* upstream, int32_t n_seg, int32_t n, int64_t ld,
                             double tau, double* grad_x, double* grad_k, lkv_stream_t stream) {
    if (!(tau > 0.0)) return fail(LKV_ERR_CONTRACT, "soft_topk_vjp: tau must be positive");  // soft_topk.cpp:171
    if (n < 1 || n_seg < 1 || ld < n) return fail(LKV_ERR_CONTRACT, "soft_topk_vjp: bad extents");
    if (!density || !upstream || !grad_x || !grad_k) return fail(LKV_ERR_CONTRACT, "soft_topk_vjp: null buffer");
    SoftTopKParams p;
    memset(&p, 0, sizeof p);
    p.n_seg = n_seg;
    p.n = n;
    p.ld = ld;
    p.tau = tau;
    p.density = const_cast<double*>(density);
    p.upstream = upstream;
    p.grad_x = grad_x;
    p.grad_k = grad_k;
    LKV_CUDA(launch_soft_topk_vjp(p, (cudaStream_t)stream), "soft topk vjp");
    return LKV_OK;
}

// ---- masked attention (training) -------------------------------------------
static lkv_status check_attn(const lkv_attn_desc* a) {
    if (!a) return fail(LKV_ERR_CONTRACT, "attention descriptor is null");
    if (a->batch < 1 || a->n_q_heads < 1 || a->n_kv_heads < 1 || a->t_q < 1 || a->t_k < 1 || a->head_dim < 1)
        return fail(LKV_ERR_CONTRACT, "attention: empty extents");  // attention.cpp:34
    if (a->n_q_heads % a->n_kv_heads) return fail(LKV_ERR_CONTRACT, "attention: n_q_heads must be a multiple of n_kv_heads");
    if (a->causal && a->query_pos_offset + 1 < 1)
        return fail(LKV_ERR_CONTRACT, "attention: first query row admits no key");  // attention.cpp:43
    if (!std::isfinite(a->scale)) return fail(LKV_ERR_CONTRACT, "attention: scale must be finite");
    if (a->dtype == LKV_BF16) {
        if (a->head_dim != 128) return fail(LKV_ERR_UNSUPPORTED, "bf16 masked attention needs head_dim 128");
    } else if (a->dtype == LKV_F32) {
        if (a->head_dim > 256 || (size_t)(a->head_dim + a->t_k) * 4 > 200 * 1024)
            return fail(LKV_ERR_UNSUPPORTED, "fp32 masked attention: head_dim <= 256 and t_k <= ~51000");
    } else {
        return fail(LKV_ERR_CONTRACT, "unknown dtype");
    }
    const int64_t rows_q = (int64_t)a->batch * a->n_q_heads * a->t_q, rows_k = (int64_t)a->batch * a->n_kv_heads * a->t_k;
    if (rows_q >= (int64_t(1) << 31) || rows_k >= (int64_t(1) << 31)) return fail(LKV_ERR_CONTRACT, "attention: too many rows");
    return LKV_OK;
}

static AttnParams attn_params(const lkv_attn_desc* a, const void* q, const void* k, const void* v, const float* mask,
                              void* ws) {
    AttnParams p;
    memset(&p, 0, sizeof p);
    p.batch = a->batch;
    p.n_q_heads = a->n_q_heads;
    p.n_kv_heads = a->n_kv_heads;
    p.t_q = a->t_q;
    p.t_k = a->t_k;
    p.causal = a->causal != 0;
    p.pos_offset = a->query_pos_offset;
    p.self_keep = a->self_always_retained != 0;
    p.scale = (float)a->scale;
    p.q = q;
    p.k = k;
    p.v = v;
    p.mask = mask;
    p.err = at<ErrWord>(ws, 0);
    return p;
}

// workspace: [error latch | D = rowsum(dO * O) (backward)]
size_t lkv_attn_workspace_bytes(const lkv_attn_desc* a) {
    if (check_attn(a)) return 0;
    return 256 + align_up(sizeof(float) * (size_t)a->batch * a->n_q_heads * a->t_q);
}

lkv_status lkv_masked_attention_fwd(const lkv_attn_desc* a, const void* q, const void* k, const void* v,
                                    const float* mask, void* out, float* lse, void* ws, size_t ws_bytes,
                                    lkv_stream_t stream) {
    lkv_status st = check_attn(a);
    if (st) return st;
    if (!q || !k || !v || !out || !lse) return fail(LKV_ERR_CONTRACT, "attention: null buffer");
    if ((st = check_ws(ws, ws_bytes, lkv_attn_workspace_bytes(a)))) return st;
    AttnParams p = attn_params(a, q, k, v, mask, ws);
    p.out = out;
    p.lse = lse;
    CUtensorMap mk, mv, mq;
    if (a->dtype == LKV_BF16) {
        const uint64_t rk = (uint64_t)a->batch * a->n_kv_heads * a->t_k, rq = (uint64_t)a->batch * a->n_q_heads * a->t_q;
        if ((st = make_map_bf16(&mk, k, 128, rk, 128)) || (st = make_map_bf16(&mv, v, 128, rk, 128)) ||
            (st = make_map_bf16(&mq, q, 128, rq, 128)))
            return st;
    }
    LKV_CUDA(launch_attn_fwd(p, a->dtype, a->head_dim, &mk, &mv, &mq, (cudaStream_t)stream), "masked attention fwd");
    return LKV_OK;
}

lkv_status lkv_masked_attention_bwd(const lkv_attn_desc* a, const void* q, const void* k, const void* v,
                                    const float* mask, const void* out, const float* lse, const void* d_out, float* dq,
                                    float* dk, float* dv, float* dmask, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    lkv_status st = check_attn(a);
    if (st) return st;
    if (!q || !k || !v || !out || !lse || !d_out || !dq || !dk || !dv) return fail(LKV_ERR_CONTRACT, "attention vjp: null buffer");
    if (mask && !dmask) return fail(LKV_ERR_CONTRACT, "attention vjp: a masked call needs dmask");
    if ((st = check_ws(ws, ws_bytes, lkv_attn_workspace_bytes(a)))) return st;
    AttnParams p = attn_params(a, q, k, v, mask, ws);
    p.out = const_cast<void*>(out);
    p.lse = const_cast<float*>(lse);
    p.dout = d_out;
    p.dsum = at<float>(ws, 256);
    p.dq = dq;
    p.dk = dk;
    p.dv = dv;
    p.dmask = mask ? dmask : nullptr;
    CUtensorMap m[8];
    if (a->dtype == LKV_BF16) {
        const uint64_t rk = (uint64_t)a->batch * a->n_kv_heads * a->t_k, rq = (uint64_t)a->batch * a->n_q_heads * a->t_q;
        if ((st = make_map_bf16(&m[0], q, 128, rq, 128)) || (st = make_map_bf16(&m[1], d_out, 128, rq, 128)) ||
            (st = make_map_bf16(&m[2], k, 128, rk, 64)) || (st = make_map_bf16(&m[3], v, 128, rk, 64)) ||
            (st = make_map_bf16(&m[4], k, 128, rk, 128)) || (st = make_map_bf16(&m[5], v, 128, rk, 128)) ||
            (st = make_map_bf16(&m[6], q, 128, rq, 64)) || (st = make_map_bf16(&m[7], d_out, 128, rq, 64)))
            return st;
    }
    LKV_CUDA(launch_attn_bwd(p, a->dtype, a->head_dim, m, (cudaStream_t)stream), "masked attention bwd");
    return LKV_OK;
}

lkv_status lkv_rope_table(int32_t t_max, int32_t head_dim, double base, int32_t pos_offset, void* table,
                          lkv_stream_t stream) {
    if (t_max < 1 || head_dim < 2 || head_dim % 2 || !(base > 0.0) || pos_offset < 0 || !table)
        return fail(LKV_ERR_CONTRACT, "rope: bad table arguments (head_dim must be even)");  // tensor.cpp:588
    LKV_CUDA(launch_rope_table(t_max, head_dim, base, pos_offset, static_cast<float2*>(table), (cudaStream_t)stream),
             "rope table");
    return LKV_OK;
}

lkv_status lkv_rope_pack(const void* k_lin, const void* v_lin, const lkv_cache_desc* layer, const void* table,
                         void* k_out, void* v_out, lkv_stream_t stream) {
    lkv_status st = check_cache(layer, false);
    if (st) return st;
    if (layer->n_layers != 1) return fail(LKV_ERR_CONTRACT, "rope_pack: one layer per call");
    if (!k_lin || !v_lin || !table || !k_out || !v_out) return fail(LKV_ERR_CONTRACT, "rope_pack: null buffer");
    if ((reinterpret_cast<uintptr_t>(k_lin) | reinterpret_cast<uintptr_t>(v_lin) | reinterpret_cast<uintptr_t>(k_out) |
         reinterpret_cast<uintptr_t>(v_out)) & 15)
        return fail(LKV_ERR_CONTRACT, "rope_pack: buffers must be 16-byte aligned");
    LKV_CUDA(launch_rope_pack(k_lin, v_lin, layer->n_seq, (int)layer->max_tokens, layer->seq_lens, layer->n_kv_heads,
                              layer->head_dim, layer->dtype, static_cast<const float2*>(table), k_out, v_out,
                              (cudaStream_t)stream),
             "rope pack");
    return LKV_OK;
}

lkv_status lkv_kv_project(const void* h, int32_t d_model, const void* wkv_t, const lkv_cache_desc* layer,
                          const void* table, void* k_out, void* v_out, lkv_stream_t stream) {
    lkv_status st = check_cache(layer, false);
    if (st) return st;
    if (layer->n_layers != 1) return fail(LKV_ERR_CONTRACT, "kv_project: one layer per call");
    if (layer->dtype != LKV_BF16 || layer->head_dim != 128)
        return fail(LKV_ERR_UNSUPPORTED, "kv_project: bf16 and head_dim 128 (tcgen05 tiles)");
    if (d_model < 64 || d_model % 64) return fail(LKV_ERR_UNSUPPORTED, "kv_project: d_model must be a multiple of 64");
    if (!h || !wkv_t || !table || !k_out || !v_out) return fail(LKV_ERR_CONTRACT, "kv_project: null buffer");
    if ((reinterpret_cast<uintptr_t>(k_out) | reinterpret_cast<uintptr_t>(v_out) |
         reinterpret_cast<uintptr_t>(table)) & 15)
        return fail(LKV_ERR_CONTRACT, "kv_project: outputs and table must be 16-byte aligned");
    KvProjParams p;
    memset(&p, 0, sizeof p);
    p.T = (int32_t)layer->max_tokens;
    p.H = layer->n_kv_heads;
    p.D = layer->head_dim;
    p.M = layer->n_seq * p.T;
    p.N = 2 * p.H * p.D;
    p.K = d_model;
    p.table = static_cast<const float2*>(table);
    p.k_out = k_out;
    p.v_out = v_out;
    if (p.N % 256) return fail(LKV_ERR_UNSUPPORTED, "kv_project: 2 * n_kv_heads * head_dim must be a multiple of 256");
    CUtensorMap ma, mb;
    if ((st = make_map_bf16(&ma, h, (uint64_t)d_model, (uint64_t)p.M, 128))) return st;
    if ((st = make_map_bf16(&mb, wkv_t, (uint64_t)d_model, (uint64_t)p.N, 128))) return st;  // a CTA's half of N
    LKV_CUDA(launch_kv_project(p, ma, mb, num_sms(), (cudaStream_t)stream), "kv project");
    return LKV_OK;
}

size_t lkv_decode_workspace_bytes(const lkv_ragged_desc* r, int32_t G) {
    if (!r || G < 1) return 0;
    return decode_layout(r, G).total;
}

lkv_status lkv_decode_plan_ex(const lkv_ragged_desc* r, int32_t rows_per_item, void* ws, size_t ws_bytes,
                              lkv_stream_t stream) {
    if (!r || !r->offsets || r->n_heads < 1) return fail(LKV_ERR_CONTRACT, "bad ragged descriptor");
    if (rows_per_item != 0 && (rows_per_item < kDecMinCh || rows_per_item > 1024 || rows_per_item % 64))
        return fail(LKV_ERR_CONTRACT, "decode plan: rows_per_item must be 0 or a multiple of 64 in [128, 1024]");
    const DecodeWs w = decode_layout(r, 1);
    lkv_status st = check_ws(ws, ws_bytes, w.items + sizeof(DecodeItem) * (size_t)w.max_items);
    if (st) return st;
    // one all-layer launch walks every item: aim for ~4 items per resident CTA; G unknown here, so
    // the combine bound assumes the largest group (16)
    LKV_CUDA(launch_decode_plan(r->offsets, r->n_heads, 1, 1, at<DecodeItem>(ws, w.items), at<int32_t>(ws, w.item_base),
                                at<int32_t>(ws, w.layer_begin), at<int32_t>(ws, w.n_items), at<int32_t>(ws, w.ch),
                                8 * num_sms(), 16, rows_per_item, (cudaStream_t)stream),
             "decode plan");
    return LKV_OK;
}

lkv_status lkv_decode_plan_info(const lkv_ragged_desc* r, const void* ws, int32_t* n_items, int32_t* rows_per_item,
                                lkv_stream_t stream) {
    if (!r || !ws) return fail(LKV_ERR_CONTRACT, "decode plan info: null argument");
    const DecodeWs w = decode_layout(r, 1);  // the plan words do not depend on G
    int32_t v[2] = {0, 0};
    LKV_CUDA(cudaMemcpyAsync(&v[0], static_cast<const char*>(ws) + w.n_items, 4, cudaMemcpyDeviceToHost,
                             (cudaStream_t)stream), "plan info");
    LKV_CUDA(cudaMemcpyAsync(&v[1], static_cast<const char*>(ws) + w.ch, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
             "plan info");
    LKV_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "plan info");
    if (n_items) *n_items = v[0];
    if (rows_per_item) *rows_per_item = v[1];
    return LKV_OK;
}

lkv_status lkv_decode_plan(const lkv_ragged_desc* r, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    return lkv_decode_plan_ex(r, 0, ws, ws_bytes, stream);
}

lkv_status lkv_decode_step(const lkv_ragged_desc* r, int32_t n_seq, int32_t n_layers, int32_t n_kv_heads,
                           int32_t n_q_heads, const void* q, const void* new_k, const void* new_v,
                           int32_t* tokens_seen, void* out, double scale, void* ws, size_t ws_bytes,
                           lkv_stream_t stream) {
    if (n_seq < 1 || n_layers < 1 || n_kv_heads < 1 || n_q_heads < n_kv_heads || n_q_heads % n_kv_heads)
        return fail(LKV_ERR_CONTRACT, "decode: n_q_heads must be a positive multiple of n_kv_heads");
    const int64_t H = (int64_t)n_seq * n_layers * n_kv_heads;
    lkv_status st = check_ragged(r, H, r ? r->head_dim : 0, r ? r->dtype : 0, true);
    if (st) return st;
    if (!q || !new_k || !new_v || !tokens_seen || !out) return fail(LKV_ERR_CONTRACT, "decode: null buffer");
    if (!(scale > 0.0) || !std::isfinite(scale)) return fail(LKV_ERR_CONTRACT, "decode: scale must be positive");
    const int G = n_q_heads / n_kv_heads;
    if (r->dtype == LKV_BF16 && (r->head_dim != 128 || G > 16))
        return fail(LKV_ERR_UNSUPPORTED, "bf16 decode needs head_dim 128 and group size <= 16");
    if (r->dtype == LKV_F32 && (size_t)G * (r->head_dim + 1024) * 4 > 200 * 1024)
        return fail(LKV_ERR_UNSUPPORTED, "fp32 decode: group too large");
    const DecodeWs w = decode_layout(r, G);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    DecodeParams p;
    memset(&p, 0, sizeof p);
    p.n_heads = (int)H;
    p.n_kv_heads = n_kv_heads;
    p.n_q_heads = n_q_heads;
    p.G = G;
    p.head_dim = r->head_dim;
    p.n_seq = n_seq;
    p.n_layers = n_layers;
    p.layer0 = 0;
    p.q_layers = n_layers;
    p.item_lo = at<int32_t>(ws, w.layer_begin);  // layer_begin[0] == 0 for every plan
    p.item_hi = at<int32_t>(ws, w.n_items);
    p.ch = at<int32_t>(ws, w.ch);
    p.out_nbt = 0;
    p.max_items = (int32_t)w.max_items;
    p.scale_log2 = (float)(scale * 1.4426950408889634);
    p.offsets = r->offsets;
    p.lens = r->lens;
    p.positions = r->positions;
    p.keys = r->keys;
    p.values = r->values;
    p.q = q;
    p.new_k = new_k;
    p.new_v = new_v;
    p.tokens_seen = tokens_seen;
    p.out = out;
    p.items = at<DecodeItem>(ws, w.items);
    p.item_base = at<int32_t>(ws, w.item_base);
    p.part_m = at<float>(ws, w.part_m);
    p.part_l = at<float>(ws, w.part_l);
    p.part_o = at<float>(ws, w.part_o);
    p.new_len = at<int32_t>(ws, w.new_len);
    p.err = at<ErrWord>(ws, w.err);
    CUtensorMap mk, mv;
    if (r->dtype == LKV_BF16) {
        if ((st = make_map_bf16(&mk, r->keys, 128, (uint64_t)r->capacity_rows, 64))) return st;
        if ((st = make_map_bf16(&mv, r->values, 128, (uint64_t)r->capacity_rows, 64))) return st;
    }
    LKV_CUDA(launch_decode(p, r->dtype, &mk, &mv, num_sms(), (cudaStream_t)stream), "decode");
    return LKV_OK;
}

// ---- fp64 reference-precision operators (the declaration-compatible include/lkv API) ------------
lkv_status lkv_soft_topk_exact(const double* x, int32_t n, double k, double tau, double* values, double* density,
                               int32_t* permutation, double* lambda, int32_t* split_m, double* clamped_k, void* ws,
                               size_t ws_bytes, lkv_stream_t stream) {
    if (!(tau > 0.0)) return fail(LKV_ERR_CONTRACT, "soft_topk_forward: tau must be positive");  // soft_topk.cpp:112
    if (n < 1) return fail(LKV_ERR_CONTRACT, "soft_topk_forward: empty scores");               // :114
    if (n > 3072) return fail(LKV_ERR_UNSUPPORTED, "soft_topk_exact: n <= 3072");
    if (!x || !values) return fail(LKV_ERR_CONTRACT, "soft_topk_exact: null buffer");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    BudgetParams p;
    memset(&p, 0, sizeof p);
    p.logits = x;
    p.n = n;
    p.mode = LKV_BUDGET_FLOOR;
    p.n_seq = 1;
    p.seq_len[0] = 1;
    p.soft = 1;
    p.k_abs = k;
    p.tau = tau;
    p.ratios_out = values;
    p.density_out = density;
    p.perm_out = permutation;
    p.lambda_out = lambda;
    p.m_out = split_m;
    p.kc_out = clamped_k;
    p.err = at<ErrWord>(ws, 0);
    LKV_CUDA(launch_budgets(p, (cudaStream_t)stream), "soft topk exact");
    return LKV_OK;
}

lkv_status lkv_f64_gemm(int32_t M, int32_t N, int32_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C, int64_t ldc, int32_t accumulate, lkv_stream_t stream) {
    if (M < 0 || N < 0 || K < 1 || !A || !B || !C || lda < K || ldb < N || ldc < N)
        return fail(LKV_ERR_CONTRACT, "f64 gemm: bad extents");
    F64GemmParams p{M, N, K, A, lda, B, ldb, C, ldc, accumulate ? 1 : 0};
    LKV_CUDA(launch_f64_gemm(p, (cudaStream_t)stream), "f64 gemm");
    return LKV_OK;
}

lkv_status lkv_f64_rmsnorm(int32_t rows, int32_t cols, const double* x, int64_t ldx, const double* gain, double eps,
                           double* out, int64_t ldo, lkv_stream_t stream) {
    if (rows < 0 || cols < 1 || !x || !gain || !out || ldx < cols || ldo < cols || !(eps > 0.0))
        return fail(LKV_ERR_CONTRACT, "f64 rmsnorm: bad arguments");
    LKV_CUDA(launch_f64_rmsnorm(rows, cols, x, ldx, gain, eps, out, ldo, (cudaStream_t)stream), "f64 rmsnorm");
    return LKV_OK;
}

lkv_status lkv_f64_rope(int32_t rows, int32_t n_heads, int32_t head_dim, double* x, int64_t ldx, int32_t pos0,
                        double base, lkv_stream_t stream) {
    if (head_dim % 2) return fail(LKV_ERR_CONTRACT, "rope: last dim must be even");  // tensor.cpp:588
    if (rows < 0 || n_heads < 1 || head_dim < 2 || !x || ldx < (int64_t)n_heads * head_dim || pos0 < 0 || !(base > 0.0))
        return fail(LKV_ERR_CONTRACT, "f64 rope: bad arguments");
    LKV_CUDA(launch_f64_rope(rows, n_heads, head_dim, x, ldx, pos0, base, (cudaStream_t)stream), "f64 rope");
    return LKV_OK;
}

lkv_status lkv_f64_attention(const lkv_f64_attn_desc* a, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!a) return fail(LKV_ERR_CONTRACT, "attention descriptor is null");
    if (a->n_q_heads < 1 || a->n_q < 1 || a->t < 1 || a->head_dim < 1 || a->group < 1)
        return fail(LKV_ERR_CONTRACT, "attention: empty extents");  // attention.cpp:34
    if (a->head_dim > 256) return fail(LKV_ERR_UNSUPPORTED, "f64 attention: head_dim <= 256");
    if (a->causal && a->query_pos_offset + 1 < 1) return fail(LKV_ERR_CONTRACT, "attention: first query row admits no key");
    if (!a->q || !a->k || !a->v || !a->out) return fail(LKV_ERR_CONTRACT, "attention: null buffer");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    F64AttnParams p;
    memset(&p, 0, sizeof p);
    p.n_qh = a->n_q_heads;
    p.G = a->group;
    p.n_q = a->n_q;
    p.t = a->t;
    p.d = a->head_dim;
    p.q = a->q;
    p.ldq = a->ldq;
    p.k = a->k;
    p.v = a->v;
    p.ldk = a->ldkv;
    p.mask = a->mask;
    p.mask_ld = a->mask_ld;
    p.causal = a->causal;
    p.qpo = a->query_pos_offset;
    p.self_keep = a->self_always_retained;
    p.scale = a->scale;
    p.out = a->out;
    p.ldo = a->ldo;
    p.p_raw = a->p_raw;
    p.p = a->p;
    p.renorm = a->renorm;
    p.err = at<ErrWord>(ws, 0);
    LKV_CUDA(launch_f64_attention(p, (cudaStream_t)stream), "f64 attention");
    return LKV_OK;
}

lkv_status lkv_f64_swiglu(int64_t n, const double* gate, const double* up, double* out, lkv_stream_t stream) {
    if (n < 0 || !gate || !up || !out) return fail(LKV_ERR_CONTRACT, "f64 swiglu: bad arguments");
    LKV_CUDA(launch_f64_swiglu(n, gate, up, out, (cudaStream_t)stream), "f64 swiglu");
    return LKV_OK;
}

lkv_status lkv_f64_embed(const int32_t* tokens, int32_t n, const double* table, int32_t d_model, int32_t vocab,
                         double* out, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (n < 0 || d_model < 1 || vocab < 1 || !tokens || !table || !out) return fail(LKV_ERR_CONTRACT, "f64 embed: bad arguments");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    LKV_CUDA(launch_f64_embed(tokens, n, table, d_model, vocab, out, at<ErrWord>(ws, 0), (cudaStream_t)stream), "f64 embed");
    return LKV_OK;
}

lkv_status lkv_f64_split_heads(int32_t t, int32_t n_heads, int32_t head_dim, const double* x, int64_t ldx, double* out,
                               int64_t out_rows, lkv_stream_t stream) {
    if (t < 0 || n_heads < 1 || head_dim < 1 || !x || !out || ldx < (int64_t)n_heads * head_dim || out_rows < t)
        return fail(LKV_ERR_CONTRACT, "f64 split_heads: bad arguments");
    LKV_CUDA(launch_f64_split_heads(t, n_heads, head_dim, x, ldx, out, out_rows, (cudaStream_t)stream), "f64 split");
    return LKV_OK;
}

lkv_status lkv_f64_token_scores(int32_t t, int32_t head_dim, int32_t input, const double* keys, int64_t ldk,
                                const double* values, int64_t ldv, const double* w1, const double* b1, const double* w2,
                                int32_t hidden, int32_t activation, double* u, void* ws, size_t ws_bytes,
                                lkv_stream_t stream) {
    if (input != LKV_SCORER_K && input != LKV_SCORER_KV) return fail(LKV_ERR_CONTRACT, "scorer input must be K or KV");
    if (activation != LKV_ACT_SILU && activation != LKV_ACT_GELU_ERF) return fail(LKV_ERR_CONTRACT, "unknown activation");
    if (t < 0 || head_dim < 1 || hidden < 1 || !keys || !w1 || !b1 || !w2 || !u || ldk < head_dim ||
        (input == LKV_SCORER_KV && (!values || ldv < head_dim)))
        return fail(LKV_ERR_CONTRACT, "token_scores: bad arguments");
    if (f64_scorer_smem(input * head_dim, hidden) > 200 * 1024) return fail(LKV_ERR_UNSUPPORTED, "f64 scorer too large");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    F64ScorerParams p{t, head_dim, input, hidden, activation, keys, ldk, values, ldv, w1, b1, w2, u, at<ErrWord>(ws, 0)};
    LKV_CUDA(launch_f64_scorer(p, (cudaStream_t)stream), "f64 scorer");
    return LKV_OK;
}

lkv_status lkv_f64_select(const double* scores, int32_t n_heads, int32_t t, int64_t ld, const int32_t* budgets,
                          const lkv_ragged_desc* out, void* ws, size_t ws_bytes, lkv_stream_t stream) {
    if (!scores || !budgets || !out || !out->offsets || !out->lens || !out->positions || n_heads < 1 || t < 0 || ld < t)
        return fail(LKV_ERR_CONTRACT, "f64 select: bad arguments");
    if (out->n_heads != n_heads) return fail(LKV_ERR_CONTRACT, "ragged n_heads mismatch");
    lkv_status st = check_ws(ws, ws_bytes, sizeof(ErrWord));
    if (st) return st;
    F64SelectParams p{t, ld, scores, budgets, out->offsets, out->positions, out->lens, at<ErrWord>(ws, 0)};
    LKV_CUDA(launch_f64_select(p, n_heads, (cudaStream_t)stream), "f64 select");
    return LKV_OK;
}

}  // extern "C"

// ============================ full model decode step ============================
namespace {

struct MatGeom {
    int N, K, NG, KU;
    size_t bytes;
};
MatGeom mat_geom(int n_virt, int K, int dtype) {
    MatGeom m;
    m.N = n_virt;
    m.K = K;
    m.NG = (n_virt + 63) / 64;
    m.KU = (K + 127) / 128;
    m.bytes = dtype == LKV_BF16 ? (size_t)m.NG * m.KU * 16384 : (size_t)K * m.NG * 64 * 4;
    return m;
}

struct ModelGeom {
    int dm, dkv, ff, D, L, Hq, H, vocab, dtype;
    size_t esz;
    MatGeom qkv, wo, gu, down, lm;
    size_t tok_embed, final_norm, lm_head, layer0, layer_stride;
    size_t o_qkv, o_wo, o_gu, o_down, o_attn_norm, o_mlp_norm, total;
};

lkv_status check_model(const lkv_model_desc* m) {
    if (!m) return fail(LKV_ERR_CONTRACT, "model descriptor is null");
    if (m->n_layers < 1 || m->n_q_heads < 1 || m->n_kv_heads < 1 || m->head_dim < 1 || m->vocab_size < 1 ||
        m->max_seq_len < 1 || m->mlp_width < 1)
        return fail(LKV_ERR_CONTRACT, "model config: extents must be >= 1");  // model.cpp:126-129
    if (m->n_q_heads % m->n_kv_heads) return fail(LKV_ERR_CONTRACT, "model config: n_query_heads must divide by n_kv_heads");
    if (m->head_dim % 2) return fail(LKV_ERR_CONTRACT, "model config: head_dim must be even for rotary pairs");
    if (m->dtype != LKV_BF16 && m->dtype != LKV_F32) return fail(LKV_ERR_CONTRACT, "model dtype must be F32 or BF16");
    if (!(m->rope_base > 0.0) || !(m->norm_eps > 0.0)) return fail(LKV_ERR_CONTRACT, "model: rope_base and norm_eps must be > 0");
    if (m->dtype == LKV_BF16 && (m->head_dim != 128 || m->n_q_heads / m->n_kv_heads > 16))
        return fail(LKV_ERR_UNSUPPORTED, "bf16 model decode needs head_dim 128 and group size <= 16");
    if ((int64_t)m->n_q_heads * m->head_dim > 128 * 1000 || m->mlp_width > 128 * 1000)
        return fail(LKV_ERR_UNSUPPORTED, "model decode: reduction lengths above 128000 exceed the stream-K split table");
    return LKV_OK;
}

ModelGeom model_geom(const lkv_model_desc* m) {
    ModelGeom g;
    g.D = m->head_dim;
    g.L = m->n_layers;
    g.Hq = m->n_q_heads;
    g.H = m->n_kv_heads;
    g.dm = g.Hq * g.D;
    g.dkv = g.H * g.D;
    g.ff = m->mlp_width;
    g.vocab = m->vocab_size;
    g.dtype = m->dtype;
    g.esz = m->dtype == LKV_BF16 ? 2 : 4;
    g.qkv = mat_geom(g.dm + 2 * g.dkv, g.dm, g.dtype);
    g.wo = mat_geom(g.dm, g.dm, g.dtype);
    g.gu = mat_geom(64 * ((g.ff + 31) / 32), g.dm, g.dtype);
    g.down = mat_geom(g.dm, g.ff, g.dtype);
    g.lm = mat_geom(g.vocab, g.dm, g.dtype);
    size_t o = 0;
    g.tok_embed = o;
    o = align_up(o + (size_t)g.vocab * g.dm * g.esz);
    g.final_norm = o;
    o = align_up(o + (size_t)g.dm * 4);
    g.lm_head = o;
    o = align_up(o + g.lm.bytes);
    g.layer0 = o;
    size_t q = 0;
    g.o_qkv = q;
    q = align_up(q + g.qkv.bytes);
    g.o_wo = q;
    q = align_up(q + g.wo.bytes);
    g.o_gu = q;
    q = align_up(q + g.gu.bytes);
    g.o_down = q;
    q = align_up(q + g.down.bytes);
    g.o_attn_norm = q;
    q = align_up(q + (size_t)g.dm * 4);
    g.o_mlp_norm = q;
    q = align_up(q + (size_t)g.dm * 4);
    g.layer_stride = q;
    g.total = o + q * g.L;
    return g;
}

struct ModelWs {
    DecodeWs dec;
    size_t x, ss, act_h, act_attn, act_ff, q, nk, nv, part, cnt, rope, total;
    int nbt;
};
size_t act_bytes(const ModelGeom& g, int K, int B, int nbt) {
    return g.dtype == LKV_BF16 ? (size_t)((K + 127) / 128) * 8 * nbt * 256 : (size_t)B * K * 4;
}
ModelWs model_ws(const ModelGeom& g, int B, const lkv_ragged_desc* r, const lkv_model_desc* m) {
    ModelWs w;
    w.dec = decode_layout(r, g.Hq / g.H);
    w.nbt = (B + 7) / 8;
    size_t o = align_up(w.dec.total);
    w.x = o;
    o = align_up(o + (size_t)B * g.dm * 4);
    w.ss = o;
    o = align_up(o + (size_t)((g.dm + 63) / 64) * B * 4);
    w.act_h = o;
    o = align_up(o + act_bytes(g, g.dm, B, w.nbt));
    w.act_attn = o;
    o = align_up(o + act_bytes(g, g.dm, B, w.nbt));
    w.act_ff = o;
    o = align_up(o + act_bytes(g, g.ff, B, w.nbt));
    w.q = o;
    o = align_up(o + (size_t)B * g.dm * g.esz);
    w.nk = o;
    o = align_up(o + (size_t)B * g.dkv * g.esz);
    w.nv = o;
    o = align_up(o + (size_t)B * g.dkv * g.esz);
    w.part = o;
    o = align_up(o + gemv_max_grid(num_sms()) * 2 * 64 * 16 * 4);
    w.cnt = o;
    const int ng_max = std::max(std::max(g.qkv.NG, g.wo.NG), std::max(std::max(g.gu.NG, g.down.NG), g.lm.NG));
    o = align_up(o + (size_t)ng_max * 4);
    w.rope = o;
    o = align_up(o + (size_t)m->max_seq_len * (g.D / 2) * 8);
    w.total = o;
    return w;
}

lkv_status check_model_cache(const lkv_model_desc* m, const lkv_ragged_desc* r, int n_seq) {
    if (n_seq < 1 || n_seq > LKV_MODEL_MAX_SEQ) return fail(LKV_ERR_UNSUPPORTED, "model decode: 1 <= n_seq <= 16");
    return check_ragged(r, (int64_t)n_seq * m->n_layers * m->n_kv_heads, m->head_dim, m->dtype, true);
}

}  // namespace

extern "C" {

lkv_status lkv_model_validate(const lkv_model_desc* m) { return check_model(m); }

size_t lkv_model_weights_bytes(const lkv_model_desc* m) {
    if (check_model(m)) return 0;
    return model_geom(m).total;
}

lkv_status lkv_model_load_param(const lkv_model_desc* m, void* weights, int32_t param, int32_t layer, const void* src,
                                lkv_stream_t stream) {
    lkv_status st = check_model(m);
    if (st) return st;
    if (!weights || !src) return fail(LKV_ERR_CONTRACT, "load_param: null buffer");
    const ModelGeom g = model_geom(m);
    const bool per_layer = param != LKV_P_TOK_EMBED && param != LKV_P_FINAL_NORM && param != LKV_P_LM_HEAD;
    if (param < LKV_P_TOK_EMBED || param > LKV_P_LM_HEAD) return fail(LKV_ERR_CONTRACT, "load_param: unknown parameter");
    if (per_layer && (layer < 0 || layer >= g.L)) return fail(LKV_ERR_CONTRACT, "load_param: layer out of range");
    unsigned char* base = static_cast<unsigned char*>(weights);
    unsigned char* lb = base + g.layer0 + (size_t)(per_layer ? layer : 0) * g.layer_stride;
    cudaStream_t s = (cudaStream_t)stream;
    auto pack = [&](const MatGeom& mg, unsigned char* dst, int K, int cols, int mode, int off) -> lkv_status {
        LKV_CUDA(launch_pack_weight(src, g.dtype, K, cols, mode, off, mg.NG, mg.KU, dst, s), "pack weight");
        return LKV_OK;
    };
    switch (param) {
        case LKV_P_TOK_EMBED:
            LKV_CUDA(cudaMemcpyAsync(base + g.tok_embed, src, (size_t)g.vocab * g.dm * g.esz, cudaMemcpyDeviceToDevice, s),
                     "tok_embed copy");
            return LKV_OK;
        case LKV_P_FINAL_NORM:
            LKV_CUDA(launch_to_f32(src, g.dtype, g.dm, reinterpret_cast<float*>(base + g.final_norm), s), "norm");
            return LKV_OK;
        case LKV_P_ATTN_NORM:
        case LKV_P_MLP_NORM:
            LKV_CUDA(launch_to_f32(src, g.dtype, g.dm,
                                   reinterpret_cast<float*>(lb + (param == LKV_P_ATTN_NORM ? g.o_attn_norm : g.o_mlp_norm)), s),
                     "norm");
            return LKV_OK;
        case LKV_P_WQ: return pack(g.qkv, lb + g.o_qkv, g.dm, g.dm, 0, 0);
        case LKV_P_WK: return pack(g.qkv, lb + g.o_qkv, g.dm, g.dkv, 0, g.dm);
        case LKV_P_WV: return pack(g.qkv, lb + g.o_qkv, g.dm, g.dkv, 0, g.dm + g.dkv);
        case LKV_P_WO: return pack(g.wo, lb + g.o_wo, g.dm, g.dm, 0, 0);
        case LKV_P_W_GATE: return pack(g.gu, lb + g.o_gu, g.dm, g.ff, 1, 0);
        case LKV_P_W_UP: return pack(g.gu, lb + g.o_gu, g.dm, g.ff, 2, 0);
        case LKV_P_W_DOWN: return pack(g.down, lb + g.o_down, g.ff, g.dm, 0, 0);
        default: return pack(g.lm, base + g.lm_head, g.dm, g.vocab, 0, 0);
    }
}

size_t lkv_model_workspace_bytes(const lkv_model_desc* m, int32_t n_seq, const lkv_ragged_desc* r) {
    if (check_model(m) || check_model_cache(m, r, n_seq)) return 0;
    return model_ws(model_geom(m), n_seq, r, m).total;
}

lkv_status lkv_model_plan_ex(const lkv_model_desc* m, const lkv_ragged_desc* r, int32_t n_seq, int32_t rows_per_item,
                             void* ws, size_t ws_bytes, lkv_stream_t stream) {
    lkv_status st = check_model(m);
    if (st || (st = check_model_cache(m, r, n_seq))) return st;
    if (rows_per_item != 0 && (rows_per_item < kDecMinCh || rows_per_item > 1024 || rows_per_item % 64))
        return fail(LKV_ERR_CONTRACT, "model plan: rows_per_item must be 0 or a multiple of 64 in [128, 1024]");
    const ModelGeom g = model_geom(m);
    const ModelWs w = model_ws(g, n_seq, r, m);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    LKV_CUDA(cudaMemsetAsync(ws, 0, w.total, s), "workspace clear");
    // per-layer launches: one wave of work items per layer (bf16), ~2 items per resident CTA (fp32)
    LKV_CUDA(launch_decode_plan(r->offsets, n_seq, g.L, g.H, at<DecodeItem>(ws, w.dec.items),
                                at<int32_t>(ws, w.dec.item_base), at<int32_t>(ws, w.dec.layer_begin),
                                at<int32_t>(ws, w.dec.n_items), at<int32_t>(ws, w.dec.ch),
                                g.dtype == LKV_BF16 ? -decode_resident_ctas(g.Hq / g.H, num_sms()) : 4 * num_sms(),
                                g.Hq / g.H, rows_per_item, s),
             "decode plan");
    LKV_CUDA(launch_rope_table(m->max_seq_len, g.D, m->rope_base, 0, at<float2>(ws, w.rope), s), "rope table");
    return LKV_OK;
}

lkv_status lkv_model_plan(const lkv_model_desc* m, const lkv_ragged_desc* r, int32_t n_seq, void* ws, size_t ws_bytes,
                          lkv_stream_t stream) {
    return lkv_model_plan_ex(m, r, n_seq, 0, ws, ws_bytes, stream);
}

lkv_status lkv_model_decode_step(const lkv_model_desc* m, const void* weights, const lkv_ragged_desc* r, int32_t n_seq,
                                 const int32_t* tokens, int32_t* tokens_seen, float* logits, void* ws, size_t ws_bytes,
                                 lkv_stream_t stream) {
    lkv_status st = check_model(m);
    if (st || (st = check_model_cache(m, r, n_seq))) return st;
    if (!weights || !tokens || !tokens_seen || !logits) return fail(LKV_ERR_CONTRACT, "model decode: null buffer");
    const ModelGeom g = model_geom(m);
    const ModelWs w = model_ws(g, n_seq, r, m);
    if ((st = check_ws(ws, ws_bytes, w.total))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int B = n_seq, G = g.Hq / g.H, sms = num_sms();
    const unsigned char* wb = static_cast<const unsigned char*>(weights);
    ErrWord* err = at<ErrWord>(ws, w.dec.err);
    float* x = at<float>(ws, w.x);
    float* ss = at<float>(ws, w.ss);

    GemvParams gp;
    memset(&gp, 0, sizeof gp);
    gp.B = B;
    gp.nbt = g.dtype == LKV_BF16 ? w.nbt : 0;
    gp.part = at<float>(ws, w.part);
    gp.cnt = at<uint32_t>(ws, w.cnt);
    gp.err = err;
    gp.dm = g.dm;
    gp.dkv = g.dkv;
    gp.head_dim = g.D;
    gp.max_seq = m->max_seq_len;
    gp.q_out = at<void>(ws, w.q);
    gp.k_out = at<void>(ws, w.nk);
    gp.v_out = at<void>(ws, w.nv);
    gp.rope = at<float2>(ws, w.rope);
    gp.tokens_seen = tokens_seen;
    gp.x = x;
    gp.ss_part = ss;
    gp.nbt_out = gp.nbt;
    gp.act_out = at<void>(ws, w.act_ff);
    gp.ff = g.ff;
    // each GEMV CTA also warms the 4 weight units after its ring's first stages in L2 before
    // griddepcontrol.wait (profiles/r02/xp_l2ahead*.sh: -0.3% per step; 8 units slower; Wo alone
    // slower, every GEMV but Wo no better than none)
    gp.l2_ahead = 4;
    auto gemv = [&](const MatGeom& mg, const unsigned char* wp, int epi, const void* act, int n_real,
                    auto&& tweak) -> cudaError_t {
        GemvParams q = gp;
        tweak(q);
        q.w = wp;
        q.NG = mg.NG;
        q.KU = mg.KU;
        q.N = n_real;
        q.K = mg.K;
        q.act = act;
        q.epi = epi;
        return launch_gemv(q, g.dtype, sms, s);
    };

    DecodeParams dp;
    memset(&dp, 0, sizeof dp);
    dp.n_heads = B * g.L * g.H;
    dp.n_kv_heads = g.H;
    dp.n_q_heads = g.Hq;
    dp.G = G;
    dp.head_dim = g.D;
    dp.n_seq = B;
    dp.n_layers = g.L;
    dp.q_layers = 1;
    dp.max_items = (int32_t)w.dec.max_items;
    dp.out_nbt = g.dtype == LKV_BF16 ? w.nbt : 0;
    dp.scale_log2 = (float)(1.0 / std::sqrt((double)g.D) * 1.4426950408889634);  // model.cpp:223
    dp.offsets = r->offsets;
    dp.lens = r->lens;
    dp.positions = r->positions;
    dp.keys = r->keys;
    dp.values = r->values;
    dp.q = at<void>(ws, w.q);
    dp.new_k = at<void>(ws, w.nk);
    dp.new_v = at<void>(ws, w.nv);
    dp.tokens_seen = tokens_seen;
    dp.out = at<void>(ws, w.act_attn);
    dp.items = at<DecodeItem>(ws, w.dec.items);
    dp.item_base = at<int32_t>(ws, w.dec.item_base);
    dp.ch = at<int32_t>(ws, w.dec.ch);
    dp.part_m = at<float>(ws, w.dec.part_m);
    dp.part_l = at<float>(ws, w.dec.part_l);
    dp.part_o = at<float>(ws, w.dec.part_o);
    dp.new_len = at<int32_t>(ws, w.dec.new_len);
    dp.err = err;
    dp.early_kv = g.dtype == LKV_BF16 ? 1 : 0;  // the step's first launch (embed) is fully serialised
    dp.lens_deferred = 1;                        // advanced by the lm_head GEMV below
    CUtensorMap mk, mv;
    if (g.dtype == LKV_BF16) {
        if ((st = make_map_bf16(&mk, r->keys, 128, (uint64_t)r->capacity_rows, 64))) return st;
        if ((st = make_map_bf16(&mv, r->values, 128, (uint64_t)r->capacity_rows, 64))) return st;
    }
    int32_t* lbeg = at<int32_t>(ws, w.dec.layer_begin);

    // rmsnorm is folded into its neighbours (model.cpp:48-53): the producer of x (embed, or the
    // residual epilogue of wo / down) also writes x * gain of the next norm as the next GEMV's
    // activations, and that GEMV scales its outputs by 1 / rms from the per-group sums of squares.
    auto norm_gain = [&](int l, bool mlp) -> const float* {
        if (l == g.L) return reinterpret_cast<const float*>(wb + g.final_norm);
        const unsigned char* lw = wb + g.layer0 + (size_t)l * g.layer_stride;
        return reinterpret_cast<const float*>(lw + (mlp ? g.o_mlp_norm : g.o_attn_norm));
    };
    void* act_h = at<void>(ws, w.act_h);
    LKV_CUDA(launch_embed(wb + g.tok_embed, g.dtype, tokens, B, g.dm, g.vocab, tokens_seen, m->max_seq_len, x, ss,
                          norm_gain(0, false), act_h, w.nbt, err, s),
             "embed");
    gp.ss_in = nullptr;
    gp.norm_dm = g.dm;
    gp.norm_eps = (float)m->norm_eps;
    gp.act_next = act_h;
    auto normed = [&](GemvParams& q) { q.ss_in = ss; };
    for (int l = 0; l < g.L; ++l) {
        const unsigned char* lw = wb + g.layer0 + (size_t)l * g.layer_stride;
        LKV_CUDA(gemv(g.qkv, lw + g.o_qkv, EPI_QKV, act_h, g.dm + 2 * g.dkv, normed), "qkv");
        dp.layer0 = l;
        dp.item_lo = lbeg + l;
        dp.item_hi = lbeg + l + 1;
        LKV_CUDA(launch_decode(dp, g.dtype, &mk, &mv, sms, s), "attention");
        const float* g_mlp = norm_gain(l, true);
        LKV_CUDA(gemv(g.wo, lw + g.o_wo, EPI_RESID, at<void>(ws, w.act_attn), g.dm,
                      [&](GemvParams& q) { q.gain_next = g_mlp; }),
                 "wo");
        LKV_CUDA(gemv(g.gu, lw + g.o_gu, EPI_SWIGLU, act_h, g.ff, normed), "gate/up");
        const float* g_next = norm_gain(l + 1, false);
        LKV_CUDA(gemv(g.down, lw + g.o_down, EPI_RESID, at<void>(ws, w.act_ff), g.dm,
                      [&](GemvParams& q) { q.gain_next = g_next; }),
                 "down");
    }
    GemvParams q = gp;
    q.f_out = logits;
    {
        q.w = wb + g.lm_head;
        q.NG = g.lm.NG;
        q.KU = g.lm.KU;
        q.N = g.vocab;
        q.K = g.dm;
        q.act = act_h;
        q.epi = EPI_F32;
        q.ss_in = ss;  // final_norm's 1 / rms
        q.lens_inc = r->lens;  // the step's deferred bookkeeping: every head + 1 row, every sequence + 1 token
        q.n_lens = dp.n_heads;
        q.seen_inc = tokens_seen;
        q.n_seen = B;
        LKV_CUDA(launch_gemv(q, g.dtype, sms, s), "lm_head");
    }
    return LKV_OK;
}

}  // extern "C"
