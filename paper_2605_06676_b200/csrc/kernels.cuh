// kernels.cuh -- launch parameter structs and host launchers of the sm_100a kernels
// (one definition shared by every translation unit).
#pragma once

#include "common.cuh"

namespace lkv_dev {
// process-wide count of kernel launches issued by this library
void note_launches(int n);
uint64_t launch_count();
// ---- budgets.cu (K2)
struct BudgetParams {
    const double* logits;
    int32_t n;
    int32_t mode;
    double R;
    int32_t n_seq;
    int32_t slack;
    double* ratios_out;
    const double* ratios_in;  // non-null: skip the solve, freeze these ratios
    int32_t* budgets_out;
    int64_t* offsets_out;
    ErrWord* err;
    // head shard (local_count > 0): this rank owns flat heads [local_begin, local_begin +
    // local_count) of every sequence; budgets_local_out gets them contiguously
    // ([n_seq][local_count]) and the offsets are scanned over the local heads only.
    int32_t local_begin;
    int32_t local_count;
    int32_t* budgets_local_out;
    const int32_t* local_ids;  // non-null: the owned heads are this list (device) instead of a range
    // soft = 1: soft_topk_forward / solve_threshold (soft_topk.cpp:58-164) with k and tau given:
    // the solve runs on logits / tau, values go to ratios_out, nothing is frozen
    int32_t soft;
    double k_abs, tau;
    double* lambda_out;
    int32_t* m_out;
    double* kc_out;
    double* density_out;
    int32_t* perm_out;
    int32_t seq_len[LKV_MAX_SEQ];
};
cudaError_t launch_budgets(const BudgetParams& p, cudaStream_t stream);
cudaError_t launch_offsets(const int32_t* budgets, int n_heads, int slack, int64_t* offsets, cudaStream_t stream);
// ---- score.cu (K1)
struct ScoreParams {
    SeqTable seq;
    int32_t in_mode, act, hidden, stride_layer, stride_head;
    const void* keys;
    const void* values;
    const void* w1t;
    const float* b1;
    const float* w2;
    float* scores;
    uint32_t* hist;  // nullable: fused top-11-bit histogram per head (tcgen05 path; zeroed by the caller)
    ErrWord* err;
    // 1: launched as the programmatic-dependent secondary of K2 on the same stream (lkv_evict):
    // it starts while K2 runs and waits for K2 before completing
    int32_t pdl;
    int32_t tile_base[LKV_MAX_SEQ + 1];
};
cudaError_t launch_score_simt(ScoreParams p, int dtype, int num_sms, cudaStream_t stream);
cudaError_t launch_score_tc(ScoreParams p, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mw,
                            int num_sms, cudaStream_t stream);
bool score_tc_supported(int dtype, int head_dim, int hidden, int in_mode);
size_t score_simt_smem_bytes(int in, int hidden);
// ---- select.cu (K3 + K4)
struct HeadSel {  // per-head top-k result of select_plan_kernel, read by the emit pass
    uint32_t mode, key_t, need_eq, pad;
};
struct SelectParams {
    SeqTable seq;
    const float* scores;
    const int32_t* budgets;
    uint32_t* hist;
    HeadSel* state;
    uint32_t* chunk_out;
    uint32_t* chunk_eqb;
    uint32_t* cands;
    const int64_t* offsets;
    int32_t* out_pos;
    int32_t* out_lens;
    const void* keys;
    const void* values;
    void* out_keys;
    void* out_values;
    int32_t row_bytes;
    int32_t gather;
    int32_t hist_ready;  // the scorer already produced `hist` (fused pass 1)
    ErrWord* err;
    int32_t chunk_base[LKV_MAX_SEQ + 1];
};
struct CompactParams {
    SeqTable seq;
    const int64_t* offsets;
    const int32_t* lens;
    const int32_t* positions;
    const void* keys;
    const void* values;
    void* out_keys;
    void* out_values;
    int32_t row_bytes;
    ErrWord* err;
};
cudaError_t launch_select(SelectParams p, int n_heads, cudaStream_t stream);
// cache_from_trace by a device mask scan (model.cpp:289-315)
struct TraceParams {
    SeqTable seq;
    const int32_t* masks;  // [n_heads][mask_ld], nonzero = keep
    int64_t mask_ld;
    uint32_t* chunk_cnt;   // [chunks] (workspace): counts, then exclusive bases within the head
    int32_t* counts;       // [n_heads] kept rows per head (the ragged lens)
    const int64_t* offsets;
    int64_t capacity;
    int32_t* out_pos;
    const void* keys;
    const void* values;
    void* out_keys;
    void* out_values;
    int32_t row_bytes;
    int32_t gather;
    ErrWord* err;
    int32_t chunk_base[LKV_MAX_SEQ + 1];
};
cudaError_t launch_trace_counts(TraceParams p, int n_heads, cudaStream_t stream);
cudaError_t launch_trace_emit(TraceParams p, cudaStream_t stream);
cudaError_t launch_compact(const CompactParams& p, int n_heads, cudaStream_t stream);
// ---- decode.cu (K5)
// Packed activation layout read by the weight-streaming GEMV (model.cu): the bf16 B operand of
// mma.m16n8k16 (k = feature, n = batch), one 8-byte fragment per lane per (16-feature step,
// 8-row batch tile).  Element (b, k) -> index in bf16 elements.
__host__ __device__ __forceinline__ size_t act_index(int b, int k, int nbt) {
    const int s = k >> 4, kk = k & 15, bt = b >> 3, g = b & 7;
    const int lane = g * 4 + ((kk & 7) >> 1);
    return (((size_t)s * nbt + bt) * 32 + lane) * 4 + (size_t)(kk >> 3) * 2 + (kk & 1);
}

struct DecodeItem {
    int32_t head, chunk;
};
struct DecodeParams {
    int32_t n_heads, n_kv_heads, n_q_heads, G, head_dim;
    int32_t n_seq, n_layers;    // cache geometry (flat head = (s * n_layers + l) * n_kv_heads + h)
    int32_t layer0, q_layers;   // this launch: layers [layer0, layer0 + q_layers) (q/out/new_k hold those)
    const int32_t* item_lo;     // device: first / one-past-last work item of this launch
    const int32_t* item_hi;
    int32_t max_items;          // upper bound on item_hi - item_lo (grid sizing)
    const int32_t* ch;          // device: rows per work item, chosen by the plan (64 | ch, <= 1024)
    int32_t out_nbt;            // 0: out is [qsl][Hq][D]; > 0: packed GEMV activations (q_layers == 1)
    float scale_log2;
    const int64_t* offsets;
    int32_t* lens;
    int32_t* positions;
    void* keys;
    void* values;
    const void* q;
    const void* new_k;
    const void* new_v;
    int32_t* tokens_seen;
    void* out;
    const DecodeItem* items;
    const int32_t* item_base;
    float* part_m;
    float* part_l;
    float* part_o;
    int32_t* new_len;  // [n_heads] lens + 1 as the attention kernel read it (chunk 0 writes it)
    ErrWord* err;
    // 1: the TMA producer streams this launch's K/V rows BEFORE griddepcontrol.wait (only the
    // consumers wait, for q / new k / new v).  Valid only when no kernel that may still be running
    // writes these heads' rows or lens: the model step's per-layer launches, whose step starts
    // with a fully serialised launch (lkv_model_step).
    int32_t early_kv;
    // 1: lens / tokens_seen are advanced by the step's last kernel (lkv_model_decode_step's lm_head
    // GEMV), not by the combine: nothing writes lens while the step's layers run, so the combine
    // reads a head's length and work-item range before griddepcontrol.wait
    int32_t lens_deferred;
};
// target_items > 0: the largest power-of-two ch giving at least that many items per layer;
// target_items < 0: the smallest ch (multiple of 64) whose busiest layer fits -target_items items;
// force_ch > 0 overrides both (a multiple of 64 in [kDecMinCh, 1024])
cudaError_t launch_decode_plan(const int64_t* offsets, int n_seq, int n_layers, int n_kv, DecodeItem* items,
                               int32_t* item_base, int32_t* layer_begin, int32_t* n_items, int32_t* ch,
                               int target_items, int G, int force_ch, cudaStream_t stream);
constexpr int kDecMinCh = 128;  // smallest work item the plan may choose (workspace sizing)
cudaError_t launch_decode(const DecodeParams& p, int dtype, const CUtensorMap* mk, const CUtensorMap* mv, int num_sms,
                          cudaStream_t stream);
int decode_resident_ctas(int G, int num_sms);

// ---- attn.cu (training-time multiplicative-mask attention)
struct AttnParams {
    int32_t batch, n_q_heads, n_kv_heads, t_q, t_k;
    int32_t causal, pos_offset, self_keep;
    float scale;
    const void* q;      // [batch][n_q_heads][t_q][d]
    const void* k;      // [batch][n_kv_heads][t_k][d]
    const void* v;
    const float* mask;  // [batch][n_kv_heads][t_k] or null (all ones)
    void* out;          // [batch][n_q_heads][t_q][d], input dtype
    float* lse;         // [batch][n_q_heads][t_q]: log2-domain masked log-sum-exp of scale * q.k
    const void* dout;
    float* dsum;        // [batch][n_q_heads][t_q] = rowsum(dO * O) (workspace)
    float* dq;          // fp32 gradients
    float* dk;
    float* dv;
    float* dmask;       // null when mask is null
    ErrWord* err;
};
cudaError_t launch_attn_fwd(const AttnParams& p, int dtype, int d, const CUtensorMap* mk, const CUtensorMap* mv,
                            const CUtensorMap* mq, cudaStream_t stream);
size_t attn_fwd_tc_smem();
cudaError_t launch_attn_bwd(const AttnParams& p, int dtype, int d, const CUtensorMap* maps, cudaStream_t stream);
size_t attn_dq_tc_smem();
size_t attn_dkv_tc_smem();
size_t attn_dq_smem();
size_t attn_dkv_smem();

// ---- softtopk.cu (Soft-TopK forward / VJP over many segments)
struct SoftTopKParams {
    int32_t n_seg, n;
    int64_t ld;            // row stride (elements) of every [n_seg][ld] array
    double tau, noise_scale;
    const double* x;       // scores
    const double* noise;   // nullable: x + noise_scale * noise (training_mask's Gumbel noise)
    const double* k;       // [n_seg] budgets
    double* values;
    double* density;       // nullable in the forward (the VJP's saved state)
    float* values_f32;     // nullable: the values as an fp32 attention mask
    double* lambda;        // nullable [n_seg]
    const double* upstream;  // VJP
    double* grad_x;
    double* grad_k;        // [n_seg]
    ErrWord* err;
};
cudaError_t launch_soft_topk_fwd(const SoftTopKParams& p, cudaStream_t stream);
cudaError_t launch_soft_topk_vjp(const SoftTopKParams& p, cudaStream_t stream);

// ---- model.cu (full decode step of the toy GQA model)
enum GemvEpi { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_F32 = 3 };
struct GemvParams {
    const void* w;       // bf16: packed 64-col x 128-k units [NG][KU]; f32: row-major [K][NG * 64]
    int32_t NG, KU;      // column groups of 64, k-units of 128
    int32_t split;       // > 0: cluster split-K (split CTAs per column group, DSMEM reduction)
    int32_t N, K;        // real output columns (virtual order) / reduction length
    int32_t B, nbt;      // batch rows, 8-row batch tiles of the packed activations
    const void* act;     // bf16: packed (act_index), K padded to KU * 128; f32: row-major [B][K]
    float* part;         // stream-K partials [2 * grid][64][16]
    uint32_t* cnt;       // per-group arrival counters (zero, self-resetting)
    ErrWord* err;
    int32_t epi;
    // EPI_QKV: columns [0, dm) -> q (RoPE), [dm, dm + dkv) -> new k (RoPE), then -> new v
    int32_t dm, dkv, head_dim, max_seq;
    void* q_out;
    void* k_out;
    void* v_out;
    const float2* rope;          // [max_seq][head_dim / 2] (cos, sin)
    const int32_t* tokens_seen;  // [B]: the step's absolute position
    // EPI_RESID: x[b][n] += y; ss_part[group][b] = sum over the group's columns of x^2; and, when
    // gain_next is set, the next rmsnorm's activations act_next = x * gain_next (packed bf16 /
    // row-major f32) -- its 1 / rms factor is applied by the consuming GEMV (ss_in below)
    float* x;
    float* ss_part;
    const float* gain_next;
    void* act_next;
    // any epi, when ss_in is set: y[n][b] *= 1 / sqrt(sum_g ss_in[g][b] / norm_dm + norm_eps), the
    // rmsnorm scale (model.cpp:48-53) of the activations this GEMV consumed
    const float* ss_in;
    int32_t norm_dm;
    float norm_eps;
    // EPI_SWIGLU: virtual column group g = gate cols [32g, 32g+32) then up cols [32g, 32g+32)
    void* act_out;
    int32_t nbt_out, ff;
    // EPI_F32
    float* f_out;
    // step bookkeeping (the model step's last GEMV, CTA 0, after griddepcontrol.wait): lens[i] += 1
    // for i < n_lens, tokens_seen[s] += 1 for s < n_seen (DecodeParams::lens_deferred)
    int32_t* lens_inc;
    int32_t n_lens;
    int32_t* seen_inc;
    int32_t n_seen;
    // bf16: weight units past the ring's first stages that each CTA prefetches into L2 before
    // griddepcontrol.wait (4 in the model step; more, or whole matrices, measured slower)
    int32_t l2_ahead;
};
cudaError_t launch_gemv(const GemvParams& p, int dtype, int num_sms, cudaStream_t stream);
size_t gemv_max_grid(int num_sms);
cudaError_t launch_embed(const void* tok_embed, int dtype, const int32_t* tokens, int B, int dm, int vocab,
                         const int32_t* tokens_seen, int max_seq, float* x, float* ss_part, const float* gain,
                         void* act, int nbt, ErrWord* err,
                         cudaStream_t stream);
cudaError_t launch_pack_weight(const void* src, int dtype, int K, int cols, int col_mode, int col_off, int NG, int KU,
                               void* dst, cudaStream_t stream);
cudaError_t launch_to_f32(const void* src, int dtype, int n, float* dst, cudaStream_t stream);
// ---- f64.cu (reference-precision operators behind include/lkv/*.hpp)
struct F64GemmParams {
    int32_t M, N, K;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    int32_t accumulate;  // C = C + A B (the sum is formed first, then added)
};
struct F64AttnParams {
    int32_t n_qh, G, n_q, t, d;  // query heads (kv head = h / G), query rows, keys, head width (<= 256)
    const double* q;             // row r, head h at q[r * ldq + h * d]
    int64_t ldq;
    const double* k;             // key j of kv head g at k[j * ldk + g * d]
    const double* v;
    int64_t ldk;
    const double* mask;          // nullable; kv head g's mask at mask[g * mask_ld + j]
    int64_t mask_ld;
    int32_t causal, qpo, self_keep;
    double scale;
    double* out;                 // row r, head h at out[r * ldo + h * d]
    int64_t ldo;
    double* p_raw;               // nullable [n_qh][n_q][t]
    double* p;                   // nullable [n_qh][n_q][t]
    double* renorm;              // nullable [n_qh][n_q]
    ErrWord* err;
};
struct F64ScorerParams {
    int32_t t, d, in_mode, hidden, act;
    const double* k;
    int64_t ldk;
    const double* v;
    int64_t ldv;
    const double* w1;  // [in][hidden] (the reference layout, policy.hpp:25)
    const double* b1;
    const double* w2;
    double* u;
    ErrWord* err;
};
struct F64SelectParams {
    int32_t t;
    int64_t ld;
    const double* scores;    // [n_heads][ld]
    const int32_t* budgets;  // [n_heads]
    const int64_t* offsets;  // [n_heads + 1]
    int32_t* positions;
    int32_t* lens;
    ErrWord* err;
};
cudaError_t launch_f64_gemm(const F64GemmParams& p, cudaStream_t s);
cudaError_t launch_f64_rmsnorm(int rows, int cols, const double* x, int64_t ldx, const double* gain, double eps,
                               double* out, int64_t ldo, cudaStream_t s);
cudaError_t launch_f64_rope(int rows, int n_heads, int d, double* x, int64_t ldx, int pos0, double base, cudaStream_t s);
cudaError_t launch_f64_attention(const F64AttnParams& p, cudaStream_t s);
cudaError_t launch_f64_swiglu(int64_t n, const double* gate, const double* up, double* out, cudaStream_t s);
cudaError_t launch_f64_embed(const int32_t* tokens, int n, const double* table, int dm, int vocab, double* out,
                             ErrWord* err, cudaStream_t s);
cudaError_t launch_f64_split_heads(int t, int H, int d, const double* x, int64_t ldx, double* out, int64_t T,
                                   cudaStream_t s);
size_t f64_scorer_smem(int in, int hidden);
cudaError_t launch_f64_scorer(const F64ScorerParams& p, cudaStream_t s);
cudaError_t launch_f64_select(const F64SelectParams& p, int n_heads, cudaStream_t s);
// ---- kvproj.cu (layer-by-layer prefill: K/V projections on tcgen05 with RoPE + pack fused)
struct KvProjParams {
    int32_t M, N, K;        // M = n_seq * T token rows, N = 2 * H * D, K = d_model
    int32_t T, H, D;
    const float2* table;    // [T][D / 2] (cos, sin) at absolute positions (lkv_rope_table)
    void* k_out;            // [n_seq][H][T][D] bf16
    void* v_out;
};
cudaError_t launch_kv_project(const KvProjParams& p, const CUtensorMap& ma, const CUtensorMap& mb, int num_sms,
                              cudaStream_t stream);
size_t kv_project_smem();
// ---- rope.cu (layer-by-layer prefill: K/V production)
cudaError_t launch_rope_table(int t_max, int head_dim, double base, int pos_offset, float2* cs, cudaStream_t stream);
cudaError_t launch_rope_pack(const void* k_lin, const void* v_lin, int n_seq, int t_max, const int32_t* seq_lens,
                             int H, int D, int dtype, const float2* cs, void* k_out, void* v_out, cudaStream_t stream);
}  // namespace lkv_dev
