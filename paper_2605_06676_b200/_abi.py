"""ctypes binding of the C ABI in include/lkv_b200.h (liblkv_b200.so).

The library is the product; this module only declares its structs and entry
points so the Python harness (tests, bench) can drive it with torch device
buffers.  Loading fails loudly when the library is missing -- there is no
fallback of any kind.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblkv_b200.so")

LKV_OK, CONTRACT, NUMERIC, BUDGET, OVERFLOW_GUARD, DEGENERATE_MASK, CUDA, UNSUPPORTED, NCCL = range(9)
COMM_ID_BYTES = 128
F32, BF16 = 0, 1
SILU, GELU_ERF = 0, 1
SCORER_K, SCORER_KV = 1, 2
BUDGET_FLOOR, BUDGET_EXACT = 0, 1
MAX_SEQ = 256

EXPORTED = [
    "lkv_abi_version", "lkv_launch_count", "lkv_last_error", "lkv_status_name", "lkv_device_check", "lkv_workspace_bytes",
    "lkv_workspace_init", "lkv_workspace_status", "lkv_ragged_capacity", "lkv_budgets", "lkv_freeze_budgets", "lkv_ragged_offsets",
    "lkv_score", "lkv_select", "lkv_compact", "lkv_evict", "lkv_evict_host", "lkv_rope_table", "lkv_rope_pack", "lkv_decode_workspace_bytes", "lkv_decode_plan",
    "lkv_decode_step", "lkv_model_validate", "lkv_model_weights_bytes", "lkv_model_load_param", "lkv_model_workspace_bytes", "lkv_model_plan",
    "lkv_model_decode_step", "lkv_budgets_shard", "lkv_evict_shard", "lkv_ragged_capacity_shard", "lkv_comm_get_unique_id",
    "lkv_comm_init", "lkv_comm_destroy", "lkv_comm_size", "lkv_comm_rank", "lkv_comm_allgatherv", "lkv_comm_gatherv",
    "lkv_attn_workspace_bytes", "lkv_masked_attention_fwd", "lkv_masked_attention_bwd", "lkv_soft_topk_fwd",
    "lkv_soft_topk_vjp", "lkv_evict_budgets", "lkv_mask_counts", "lkv_cache_from_trace", "lkv_decode_plan_ex",
    "lkv_model_plan_ex", "lkv_decode_plan_info", "lkv_evict_host_shard", "lkv_soft_topk_exact", "lkv_f64_gemm",
    "lkv_f64_rmsnorm", "lkv_f64_rope", "lkv_f64_attention", "lkv_f64_swiglu", "lkv_f64_embed", "lkv_f64_split_heads",
    "lkv_f64_token_scores", "lkv_f64_select", "lkv_kv_project", "lkv_budgets_heads", "lkv_evict_heads",
    "lkv_evict_host_heads",
]


class CacheDesc(C.Structure):
    _fields_ = [("n_seq", C.c_int32), ("n_layers", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("max_tokens", C.c_int64), ("dtype", C.c_int32), ("_pad", C.c_int32), ("keys", C.c_void_p),
                ("values", C.c_void_p), ("seq_lens", C.POINTER(C.c_int32))]


class ScorerDesc(C.Structure):
    _fields_ = [("input", C.c_int32), ("activation", C.c_int32), ("hidden", C.c_int32), ("n_scorers", C.c_int32),
                ("stride_layer", C.c_int32), ("stride_head", C.c_int32), ("w1t", C.c_void_p), ("b1", C.c_void_p),
                ("w2", C.c_void_p)]


class RaggedDesc(C.Structure):
    _fields_ = [("n_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32), ("decode_slack", C.c_int32),
                ("capacity_rows", C.c_int64), ("offsets", C.c_void_p), ("lens", C.c_void_p), ("keys", C.c_void_p),
                ("values", C.c_void_p), ("positions", C.c_void_p)]


class AttnDesc(C.Structure):
    _fields_ = [("batch", C.c_int32), ("n_q_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("t_q", C.c_int32),
                ("t_k", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32), ("causal", C.c_int32),
                ("query_pos_offset", C.c_int32), ("self_always_retained", C.c_int32), ("scale", C.c_double)]


class F64AttnDesc(C.Structure):
    _fields_ = [("n_q_heads", C.c_int32), ("group", C.c_int32), ("n_q", C.c_int32), ("t", C.c_int32),
                ("head_dim", C.c_int32), ("causal", C.c_int32), ("query_pos_offset", C.c_int32),
                ("self_always_retained", C.c_int32), ("scale", C.c_double), ("q", C.c_void_p), ("ldq", C.c_int64),
                ("k", C.c_void_p), ("v", C.c_void_p), ("ldkv", C.c_int64), ("mask", C.c_void_p),
                ("mask_ld", C.c_int64), ("out", C.c_void_p), ("ldo", C.c_int64), ("p_raw", C.c_void_p),
                ("p", C.c_void_p), ("renorm", C.c_void_p)]


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_q_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("vocab_size", C.c_int32), ("max_seq_len", C.c_int32), ("mlp_width", C.c_int32), ("dtype", C.c_int32),
                ("rope_base", C.c_double), ("norm_eps", C.c_double)]


(P_TOK_EMBED, P_WQ, P_WK, P_WV, P_WO, P_ATTN_NORM, P_MLP_NORM, P_W_GATE, P_W_UP, P_W_DOWN, P_FINAL_NORM,
 P_LM_HEAD) = range(12)
MODEL_MAX_SEQ = 16

_lib = None


def load():
    """Load liblkv_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `make -C paper_2605_06676_b200` "
                          "(or __graft_entry__.build()); there is no fallback")
    L = C.CDLL(LIB_PATH)
    vp, sz, i32, i64, dbl = C.c_void_p, C.c_size_t, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.lkv_abi_version.restype = C.c_int
    L.lkv_launch_count.restype = C.c_uint64
    L.lkv_last_error.restype = C.c_char_p
    L.lkv_status_name.restype = C.c_char_p
    L.lkv_status_name.argtypes = [C.c_int]
    L.lkv_device_check.restype = C.c_int
    L.lkv_workspace_bytes.restype = sz
    L.lkv_workspace_bytes.argtypes = [P(CacheDesc), i32]
    L.lkv_workspace_init.argtypes = [vp, sz, vp]
    L.lkv_workspace_status.argtypes = [vp, vp]
    L.lkv_ragged_capacity.restype = i64
    L.lkv_ragged_capacity.argtypes = [P(CacheDesc), dbl, i32]
    L.lkv_budgets.argtypes = [vp, i32, dbl, i32, P(i32), i32, i32, vp, vp, vp, vp, sz, vp]
    L.lkv_freeze_budgets.argtypes = [vp, i32, dbl, i32, P(i32), i32, i32, vp, vp, vp, sz, vp]
    L.lkv_ragged_offsets.argtypes = [vp, i32, i32, vp, vp]
    L.lkv_score.argtypes = [P(CacheDesc), P(ScorerDesc), vp, vp, sz, vp]
    L.lkv_select.argtypes = [P(CacheDesc), vp, vp, P(RaggedDesc), i32, vp, sz, vp]
    L.lkv_compact.argtypes = [P(CacheDesc), P(RaggedDesc), vp, sz, vp]
    L.lkv_mask_counts.argtypes = [P(CacheDesc), vp, i64, vp, vp, sz, vp]
    L.lkv_cache_from_trace.argtypes = [P(CacheDesc), vp, i64, P(RaggedDesc), vp, sz, vp]
    L.lkv_evict.argtypes = [P(CacheDesc), P(ScorerDesc), vp, dbl, i32, P(RaggedDesc), vp, vp, vp, vp, sz, vp]
    L.lkv_evict_host.argtypes = [P(CacheDesc), vp, vp, P(ScorerDesc), vp, dbl, i32, P(RaggedDesc), P(RaggedDesc), i32,
                                 vp, sz, vp]
    L.lkv_evict_host_shard.argtypes = [P(CacheDesc), vp, vp, P(ScorerDesc), vp, i32, i32, dbl, i32, P(RaggedDesc),
                                       P(RaggedDesc), i32, vp, sz, vp]
    L.lkv_evict_host_shard.restype = C.c_int
    L.lkv_soft_topk_exact.argtypes = [vp, i32, dbl, dbl, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_f64_gemm.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp, i64, i32, vp]
    L.lkv_f64_rmsnorm.argtypes = [i32, i32, vp, i64, vp, dbl, vp, i64, vp]
    L.lkv_f64_rope.argtypes = [i32, i32, i32, vp, i64, i32, dbl, vp]
    L.lkv_f64_attention.argtypes = [P(F64AttnDesc), vp, sz, vp]
    L.lkv_f64_swiglu.argtypes = [i64, vp, vp, vp, vp]
    L.lkv_f64_embed.argtypes = [vp, i32, vp, i32, i32, vp, vp, sz, vp]
    L.lkv_f64_split_heads.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp]
    L.lkv_f64_token_scores.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp, vp, vp, i32, i32, vp, vp, sz, vp]
    L.lkv_f64_select.argtypes = [vp, i32, i32, i64, vp, P(RaggedDesc), vp, sz, vp]
    for name in ["lkv_soft_topk_exact", "lkv_f64_gemm", "lkv_f64_rmsnorm", "lkv_f64_rope", "lkv_f64_attention",
                 "lkv_f64_swiglu", "lkv_f64_embed", "lkv_f64_split_heads", "lkv_f64_token_scores", "lkv_f64_select"]:
        getattr(L, name).restype = C.c_int
    L.lkv_budgets_heads.argtypes = [vp, i32, dbl, i32, P(i32), i32, i32, vp, i32, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_evict_heads.argtypes = [P(CacheDesc), P(ScorerDesc), vp, i32, vp, dbl, i32, P(RaggedDesc), vp, vp, vp, vp,
                                  sz, vp]
    L.lkv_evict_host_heads.argtypes = [P(CacheDesc), vp, vp, P(ScorerDesc), vp, i32, vp, dbl, i32, P(RaggedDesc),
                                       P(RaggedDesc), i32, vp, sz, vp]
    for name in ["lkv_budgets_heads", "lkv_evict_heads", "lkv_evict_host_heads"]:
        getattr(L, name).restype = C.c_int
    L.lkv_kv_project.argtypes = [vp, i32, vp, P(CacheDesc), vp, vp, vp, vp]
    L.lkv_kv_project.restype = C.c_int
    L.lkv_rope_table.argtypes = [i32, i32, dbl, i32, vp, vp]
    L.lkv_rope_pack.argtypes = [vp, vp, P(CacheDesc), vp, vp, vp, vp]
    L.lkv_decode_workspace_bytes.restype = sz
    L.lkv_decode_workspace_bytes.argtypes = [P(RaggedDesc), i32]
    L.lkv_decode_plan.argtypes = [P(RaggedDesc), vp, sz, vp]
    L.lkv_decode_plan_ex.argtypes = [P(RaggedDesc), i32, vp, sz, vp]
    L.lkv_decode_plan_info.argtypes = [P(RaggedDesc), vp, P(i32), P(i32), vp]
    L.lkv_decode_step.argtypes = [P(RaggedDesc), i32, i32, i32, i32, vp, vp, vp, vp, vp, dbl, vp, sz, vp]
    L.lkv_model_validate.argtypes = [P(ModelDesc)]
    L.lkv_model_weights_bytes.restype = sz
    L.lkv_model_weights_bytes.argtypes = [P(ModelDesc)]
    L.lkv_model_load_param.argtypes = [P(ModelDesc), vp, i32, i32, vp, vp]
    L.lkv_model_workspace_bytes.restype = sz
    L.lkv_model_workspace_bytes.argtypes = [P(ModelDesc), i32, P(RaggedDesc)]
    L.lkv_model_plan.argtypes = [P(ModelDesc), P(RaggedDesc), i32, vp, sz, vp]
    L.lkv_model_plan_ex.argtypes = [P(ModelDesc), P(RaggedDesc), i32, i32, vp, sz, vp]
    L.lkv_model_decode_step.argtypes = [P(ModelDesc), vp, P(RaggedDesc), i32, vp, vp, vp, vp, sz, vp]
    L.lkv_budgets_shard.argtypes = [vp, i32, dbl, i32, P(i32), i32, i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_evict_shard.argtypes = [P(CacheDesc), P(ScorerDesc), vp, i32, i32, dbl, i32, P(RaggedDesc), vp, vp, vp, vp,
                                  sz, vp]
    L.lkv_ragged_capacity_shard.restype = i64
    L.lkv_ragged_capacity_shard.argtypes = [P(CacheDesc), i32, dbl, i32]
    L.lkv_comm_get_unique_id.argtypes = [vp]
    L.lkv_comm_init.argtypes = [P(vp), vp, i32, i32]
    L.lkv_comm_destroy.argtypes = [vp]
    L.lkv_comm_size.restype = i32
    L.lkv_comm_size.argtypes = [vp]
    L.lkv_comm_rank.restype = i32
    L.lkv_comm_rank.argtypes = [vp]
    L.lkv_comm_allgatherv.argtypes = [vp, vp, vp, P(i64), P(i64), vp]
    L.lkv_comm_gatherv.argtypes = [vp, vp, vp, P(i64), P(i64), i32, vp]
    L.lkv_attn_workspace_bytes.restype = sz
    L.lkv_attn_workspace_bytes.argtypes = [P(AttnDesc)]
    L.lkv_masked_attention_fwd.argtypes = [P(AttnDesc), vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_masked_attention_bwd.argtypes = [P(AttnDesc), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_soft_topk_fwd.argtypes = [vp, vp, dbl, i32, i32, i64, vp, dbl, vp, vp, vp, vp, vp, sz, vp]
    L.lkv_soft_topk_vjp.argtypes = [vp, vp, i32, i32, i64, dbl, vp, vp, vp]
    L.lkv_evict_budgets.argtypes = [P(CacheDesc), P(ScorerDesc), vp, P(RaggedDesc), vp, vp, sz, vp]
    L.lkv_evict_budgets.restype = C.c_int
    L.lkv_soft_topk_fwd.restype = C.c_int
    L.lkv_soft_topk_vjp.restype = C.c_int
    L.lkv_masked_attention_fwd.restype = C.c_int
    L.lkv_masked_attention_bwd.restype = C.c_int
    for name in ["lkv_budgets_shard", "lkv_evict_shard", "lkv_comm_get_unique_id", "lkv_comm_init", "lkv_comm_destroy",
                 "lkv_comm_allgatherv", "lkv_comm_gatherv"]:
        getattr(L, name).restype = C.c_int
    for name in ["lkv_workspace_init", "lkv_workspace_status", "lkv_budgets", "lkv_freeze_budgets", "lkv_ragged_offsets", "lkv_score",
                 "lkv_select", "lkv_compact", "lkv_evict", "lkv_evict_host", "lkv_rope_table", "lkv_rope_pack", "lkv_decode_plan", "lkv_decode_step",
                 "lkv_model_validate", "lkv_model_load_param", "lkv_model_plan", "lkv_model_decode_step",
                 "lkv_mask_counts", "lkv_cache_from_trace", "lkv_decode_plan_ex", "lkv_model_plan_ex",
                 "lkv_decode_plan_info"]:
        getattr(L, name).restype = C.c_int
    _lib = L
    return L
