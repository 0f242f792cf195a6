// lkv_b200_dropin.hpp -- C++ host layer over the C ABI (include/lkv_b200.h) that
// mirrors the reference's hot-path API (/root/reference/proj/include/lkv) so a
// caller of the reference can switch to the B200 path by changing a namespace.
//
//   reference (lkv::, fp64 CPU)                 here (lkv::b200::, sm_100a device)
//   ------------------------------------------  -----------------------------------------
//   allocate_budgets   policy.hpp:67           allocate_budgets   (K2 on device, fp64)
//   freeze_budgets     policy.hpp:70           freeze_budgets / freeze_budgets_exact (K2)
//   token_scores       policy.hpp:73           token_scores       (K1, fp32 SIMT or bf16 tcgen05)
//   inference_select   policy.hpp:81           inference_select   (K3 on fp32 scores)
//   hard_topk          soft_topk.hpp:71        hard_topk          (K3)
//   cache_from_trace   model.hpp:99            cache_from_trace   (K4)
//   prefill_with_eviction evictsim.hpp:74      prefill_with_eviction (fused K2->K1->K3+K4, K/V given)
//   decode_step (attention block) model.hpp:95 decode_attention   (K5: append + attend)
//   kv_memory_bytes    evictsim.hpp:38-40      kv_memory_bytes
//
// Calls are synchronous (like the reference) and throw the reference's exception
// types (errors.hpp:10-32, same "kind: " message prefixes).  Inputs are host
// buffers; the device computes in fp32 (or bf16 when Precision::bf16 is asked),
// so scores/attention outputs match the reference within the tolerances of
// BASELINE.json (1e-5 fp32, 1e-2 bf16) and budgets / indices / layout are exact
// with respect to the device's own scores (stage-wise parity).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(__GNUC__)
#pragma GCC visibility push(default)  // exported from the -fvisibility=hidden library
#endif
namespace lkv::b200 {

// ---- errors (errors.hpp:10-32) ------------------------------------------------------------
struct contract_error : std::runtime_error {
    explicit contract_error(const std::string& m) : std::runtime_error("contract: " + m) {}
};
struct numeric_error : std::runtime_error {
    explicit numeric_error(const std::string& m) : std::runtime_error("numeric: " + m) {}
};
struct budget_error : std::runtime_error {
    explicit budget_error(const std::string& m) : std::runtime_error("budget: " + m) {}
};
struct overflow_guard_error : std::runtime_error {
    explicit overflow_guard_error(const std::string& m) : std::runtime_error("overflow guard: " + m) {}
};
struct degenerate_mask_error : std::runtime_error {
    explicit degenerate_mask_error(const std::string& m) : std::runtime_error("degenerate mask: " + m) {}
};
struct device_error : std::runtime_error {  // CUDA / unsupported device (no reference analogue)
    explicit device_error(const std::string& m) : std::runtime_error("device: " + m) {}
};

enum class Precision { fp32, bf16 };
enum class Activation { silu, gelu_erf };

// ---- policy.hpp:24-32: two-layer scorer in -> hidden -> 1, no output bias -----------------
struct Mlp2 {
    int in = 0, hidden = 0;
    std::vector<double> w1;  // [in x hidden] row-major
    std::vector<double> b1;  // [hidden]
    std::vector<double> w2;  // [hidden]
    int64_t param_count() const { return (int64_t)w1.size() + (int64_t)b1.size() + (int64_t)w2.size(); }
};

// ---- policy.hpp:54-63 ------------------------------------------------------------------------
struct BudgetTable {
    int n_layers = 0;
    int n_kv_heads = 0;
    double target_ratio = 0.0;
    std::vector<double> ratios;  // [L*H], entries in (0,1), sum R*L*H
    std::vector<double> logits;  // the LKV-H scores the table came from (device re-freezing)
    double at(int layer, int head) const { return ratios[(size_t)(layer * n_kv_heads + head)]; }
};

BudgetTable allocate_budgets(std::span<const double> scores, double target_ratio, int n_layers, int n_kv_heads);
std::vector<int> freeze_budgets(const BudgetTable& table, int t);
std::vector<int> freeze_budgets_exact(const BudgetTable& table, int t);
// policy.cpp:301-311 -- "layer,head,ratio" ("%.6f"), the `lkv export-budgets` budgets.csv
std::string budget_table_csv(const BudgetTable& table);

// ---- scorer / selection ------------------------------------------------------------------------
// keys, values: [t x d] row-major.  in = d (values ignored, pass empty) or 2d ([k;v]).
std::vector<double> token_scores(std::span<const double> keys, std::span<const double> values, int t, int d,
                                 const Mlp2& scorer, Activation act = Activation::silu,
                                 Precision prec = Precision::fp32);
std::vector<int> hard_topk(std::span<const float> u, int b);
std::vector<int> inference_select(std::span<const float> u, int b);

// ---- model.hpp:55-71 cache ----------------------------------------------------------------------
struct HeadCache {
    std::vector<double> keys;    // retained x d
    std::vector<double> values;  // retained x d
    std::vector<int> retained_positions;  // strictly increasing
    int retained() const { return (int)retained_positions.size(); }
};

struct KvCache {
    int n_layers = 0, n_kv_heads = 0, head_dim = 0;
    int tokens_seen = 0;
    std::vector<HeadCache> heads;  // layer-major l * n_kv_heads + h
    HeadCache& head(int l, int h) { return heads[(size_t)(l * n_kv_heads + h)]; }
    const HeadCache& head(int l, int h) const { return heads[(size_t)(l * n_kv_heads + h)]; }
};

// Dense per-head K/V of one sequence: keys[(l*H + h)] is [t x d].
struct KvTrace {
    int n_layers = 0, n_kv_heads = 0, head_dim = 0, t = 0;
    std::vector<std::vector<double>> keys, values;
};

// model.cpp:289-315: keep the rows of each head whose binary mask is set, ascending.
KvCache cache_from_trace(const KvTrace& trace, const std::vector<std::vector<int>>& hard_masks,
                         Precision prec = Precision::fp32);

// ---- evictsim.hpp:50-78 -------------------------------------------------------------------------
struct SimReport {
    std::vector<int> retained_per_head;
    double kv_bytes_full = 0.0, kv_bytes_compressed = 0.0, reduction = 0.0;
    double evict_device_seconds = 0.0;
    int64_t scoring_ops = 0;
};

// The score -> select -> compact loop of prefill_with_eviction (evictsim.cpp:161-215) for K/V
// already computed: one scorer per (layer, head) (reference layout, policy.cpp:100-102) or one
// per layer.  Budgets are validated like the reference (evictsim.cpp:104-109).
std::pair<KvCache, SimReport> prefill_with_eviction(const KvTrace& trace, const std::vector<int>& budgets,
                                                    const std::vector<Mlp2>& scorers, Activation act,
                                                    Precision prec = Precision::fp32);

// ---- model.cpp:240-265 decode attention ------------------------------------------------------------
// For every layer: append k_new/v_new [H x d] (post-RoPE) with position tokens_seen, then every
// query head qh attends over head qh / G: out = softmax(scale q K^T) V.  q: [L][Hq][d].
// Returns [L][Hq][d]; advances cache.tokens_seen.  The device keeps a resident copy of the
// cache between calls (see DecodeSession); this convenience form uploads per call.
std::vector<double> decode_attention(KvCache& cache, std::span<const double> q, int n_q_heads,
                                     std::span<const double> k_new, std::span<const double> v_new,
                                     Precision prec = Precision::fp32);

// ---- evictsim.cpp:56-81 ------------------------------------------------------------------------------
struct MemoryModel {
    int n_layers = 32, n_kv_heads = 8, head_dim = 128;
    double bytes_per_element = 2.0;
    int64_t tokens = 200000;
};
struct MemoryReport {
    double full_bytes = 0.0, compressed_bytes = 0.0, reduction_factor = 0.0;
};
MemoryReport kv_memory_bytes(const MemoryModel& model, double retention);
MemoryReport kv_memory_bytes(const MemoryModel& model, const std::vector<int>& per_head_budgets);

// ---- trained-policy ingestion (checkpoint.cpp:56-86, container.cpp:92-137) -------------------------
// LKV policy checkpoint written by the reference (`lkv train` -> lkv_params.bin).
struct LkvParams {
    int n_layers = 0, n_kv_heads = 0, d_e = 0, d_head = 0;
    std::vector<double> head_embeddings;  // [L*H x d_e]
    Mlp2 head_predictor;                  // d_e -> d_e/2 -> 1
    std::vector<Mlp2> token_scorers;      // one per (l, h): 2 d_head -> d_head -> 1
};
LkvParams load_lkv_params(const std::string& path);
// policy.cpp:106-108 -- the LKV-H logits (fp64 scorer on the device)
std::vector<double> head_scores(const LkvParams& params);
// the reference's tensor container (container.cpp:45-137): 8-byte LE metadata length, JSON
// metadata, f64 / f32 payloads; every tensor comes back as fp64
struct ContainerTensor {
    std::vector<int> shape;
    std::vector<double> v;
};
std::vector<std::pair<std::string, ContainerTensor>> read_container(const std::string& path);

// ---- training-time operators -----------------------------------------------
// soft_topk.hpp:36-44 / :60-67 -- values sum to the clamped k; the saved density terms feed the VJP.
struct SoftTopKOutput {
    std::vector<double> values;
    std::vector<double> density_terms;
    double threshold_lambda = 0.0;
    double clamped_k = 0.0;
    double tau = 1.0;
};
SoftTopKOutput soft_topk_forward(std::span<const double> x, double k, double tau);
std::pair<std::vector<double>, double> soft_topk_vjp(const SoftTopKOutput& saved, std::span<const double> upstream,
                                                     double tau);
// training_mask (policy.cpp:138-150) with the Gumbel noise supplied (scores + noise_scale * noise)
SoftTopKOutput training_mask(std::span<const double> u, double b_continuous, double tau,
                             std::span<const double> gumbel_noise, double noise_scale);

// attention.hpp:20-74 -- one head; the saved state is the device form (log2 masked LSE and the
// output the backward's D = rowsum(dO * O) reads) instead of the reference's p_raw / p matrices.
struct AttentionCall {
    int n_q = 0, t = 0, d = 0;
    std::vector<double> queries, keys, values, soft_mask;  // soft_mask empty = all ones
    bool causal = true;
    double scale = 0.0;
    int query_pos_offset = 0;
    bool self_always_retained = false;
};
struct AttentionSaved {
    std::vector<float> lse;     // [n_q], log2 domain
    std::vector<double> out;    // [n_q x d] as computed on the device (rounded to the compute dtype)
    Precision prec = Precision::fp32;
};
struct AttentionGrads {
    std::vector<double> queries, keys, values, soft_mask;  // soft_mask empty when the call had none
};
std::vector<double> masked_attention_dense(const AttentionCall& call, AttentionSaved* saved = nullptr,
                                           Precision prec = Precision::fp32);
AttentionGrads masked_attention_vjp(const AttentionCall& call, const AttentionSaved& saved,
                                    const std::vector<double>& upstream);

// Throws device_error unless an sm_100 (B200) device is current.
void require_b200();

}  // namespace lkv::b200
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
