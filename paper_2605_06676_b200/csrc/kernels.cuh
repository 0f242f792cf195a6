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
    int32_t tile_base[LKV_MAX_SEQ + 1];
};
cudaError_t launch_score_simt(ScoreParams p, int dtype, int num_sms, cudaStream_t stream);
cudaError_t launch_score_tc(ScoreParams p, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mw,
                            int num_sms, cudaStream_t stream);
bool score_tc_supported(int dtype, int head_dim, int hidden, int in_mode);
size_t score_simt_smem_bytes(int in, int hidden);
// ---- select.cu (K3 + K4)
struct HeadSel {
    uint32_t mode, bin1, rem1, n_cand, key_t, need_eq, pad[2];
};
struct SelectParams {
    SeqTable seq;
    const float* scores;
    const int32_t* budgets;
    uint32_t* hist;
    HeadSel* state;
    uint32_t* chunk_gt;
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
cudaError_t launch_compact(const CompactParams& p, int n_heads, cudaStream_t stream);
// ---- decode.cu (K5)
struct DecodeItem {
    int32_t head, chunk;
};
struct DecodeParams {
    int32_t n_heads, n_kv_heads, n_q_heads, G, head_dim;
    const int32_t* n_items;
    int32_t max_items;
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
    int32_t heads_per_seq;
    void* out;
    const DecodeItem* items;
    const int32_t* item_base;
    float* part_m;
    float* part_l;
    float* part_o;
    ErrWord* err;
};
cudaError_t launch_decode_plan(const int64_t* offsets, int n_heads, DecodeItem* items, int32_t* item_base,
                               int32_t* n_items, cudaStream_t stream);
cudaError_t launch_decode(const DecodeParams& p, int dtype, const CUtensorMap* mk, const CUtensorMap* mv, int num_sms,
                          cudaStream_t stream);
// ---- rope.cu (layer-by-layer prefill: K/V production)
cudaError_t launch_rope_table(int t_max, int head_dim, double base, int pos_offset, float2* cs, cudaStream_t stream);
cudaError_t launch_rope_pack(const void* k_lin, const void* v_lin, int n_seq, int t_max, const int32_t* seq_lens,
                             int H, int D, int dtype, const float2* cs, void* k_out, void* v_out, cudaStream_t stream);
}  // namespace lkv_dev
