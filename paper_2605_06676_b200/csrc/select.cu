// select.cu -- K3 per-head top-k (inference_select -> hard_topk, soft_topk.cpp:191-201)
// fused with K4 compaction (evictsim.cpp:202-215), plus the standalone gather.
//
// Semantics: per head keep exactly b rows, the b largest fp32 scores, ties to
// the lowest index (std::stable_sort with x[a] > x[b]); -0.0 == +0.0; NaN is a
// numeric_error; b outside [0, t] a budget_error.  Retained positions are
// written ascending (the compaction walk, evictsim.cpp:205-212).
//
// Algorithm (HBM-bound, 12 bytes/row of score traffic):
//   S1 hist     per 4096-row chunk: 2048-bin histogram of the top 11 key bits
//               (fused into K1's epilogue on the tcgen05 path)
//   S2-S4 plan  one CTA per head (select_plan_kernel):
//     S2        the bin holding the b-th largest key
//     S3        count rows above that bin per chunk; append rows inside it
//               (the candidates, usually a few % of t) to a per-head list
//     S4        radix-select the remaining 21 bits over the candidates ->
//               exact threshold key T and the number of T-equal rows still
//               needed; per-chunk output offsets by a chunk scan
//   S5 emit     per chunk: keep key > T, or key == T while the running equal
//               rank (index order) is below the need; block scans give each
//               kept row its slot; optionally gather its K/V rows (16-byte
//               vectors) straight into the ragged cache.
#include "kernels.cuh"

namespace lkv_dev {

constexpr int kChunk = 4096;
constexpr int kSelThreads = 256;
constexpr int kPerThread = kChunk / kSelThreads;  // 16 contiguous rows per thread
constexpr int kMaxChunksPerHead = 1024;           // t <= 4M rows per head

enum : uint32_t { kModeNormal = 0, kModeNone = 1, kModeAll = 2 };

// key <-> float for the float-domain compares (f32_key's inverse on keys of real floats)
constexpr uint32_t kKeyNegInf = 0x007fffffu;  // f32_key(-inf)
constexpr uint32_t kKeyPosInf = 0xff800000u;  // f32_key(+inf)
__device__ __forceinline__ float key_to_f32(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// the largest float below f (f != -0.0, f finite or +inf)
__device__ __forceinline__ float float_below(float f) {
    const uint32_t u = __float_as_uint(f);
    if (u == 0u) return __uint_as_float(0x80000001u);  // +0.0 -> -denorm_min
    return __uint_as_float((u & 0x80000000u) ? u + 1u : u - 1u);
}



struct ChunkInfo {
    int head, c, cbase, t, c0, n;  // c: chunk in head, cbase: global chunk id of head's chunk 0
};

__device__ __forceinline__ ChunkInfo decode_chunk(const SelectParams& p, int chunk) {
    int s = 0;
    while (s + 1 < p.seq.n_seq && p.chunk_base[s + 1] <= chunk) ++s;
    const int t = p.seq.len[s];
    const int cph = (t + kChunk - 1) / kChunk;
    const int local = chunk - p.chunk_base[s];
    const int hs = local / cph;
    ChunkInfo ci;
    ci.c = local - hs * cph;
    ci.head = s * p.seq.n_layers * p.seq.n_kv_heads + hs;
    ci.cbase = chunk - ci.c;
    ci.t = t;
    ci.c0 = ci.c * kChunk;
    ci.n = min(kChunk, t - ci.c0);
    return ci;
}

__device__ __forceinline__ int head_len(const SelectParams& p, int head) { return p.seq.len[head_seq(p.seq, head)]; }

// the radix keys of a thread's 16 contiguous rows [j0, j0 + 16) of a chunk (n rows): four 16-byte
// loads when the rows are all present and aligned, else guarded scalar loads (rows past n -> 0)
__device__ __forceinline__ void load_keys16(const float* sc, int j0, int n, uint32_t (&k)[kPerThread]) {
    static_assert(kPerThread == 16, "four float4 per thread");
    if (j0 + kPerThread <= n && (reinterpret_cast<uintptr_t>(sc + j0) & 15) == 0) {
        const float4* v = reinterpret_cast<const float4*>(sc + j0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 f = __ldg(v + q);
            k[4 * q + 0] = f32_key(f.x);
            k[4 * q + 1] = f32_key(f.y);
            k[4 * q + 2] = f32_key(f.z);
            k[4 * q + 3] = f32_key(f.w);
        }
    } else {
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) k[q] = (j0 + q < n) ? f32_key(sc[j0 + q]) : 0u;
    }
}

// ---- S1 --------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelThreads) select_hist_kernel(const __grid_constant__ SelectParams p) {
    __shared__ uint32_t h[2048];
    const ChunkInfo ci = decode_chunk(p, blockIdx.x);
    const int b = p.budgets[ci.head];
    if (b < 0 || b > ci.t) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_BUDGET, ci.head);
        return;
    }
    if (b == 0 || b == ci.t) return;  // resolved without a histogram
    for (int i = threadIdx.x; i < 2048; i += kSelThreads) h[i] = 0;
    __syncthreads();
    const float* sc = p.scores + (size_t)ci.head * p.seq.T + ci.c0;
    bool nan = false;
    for (int i = threadIdx.x; i < ci.n; i += kSelThreads) {
        const float f = sc[i];
        nan |= f32_is_nan(f);
        atomicAdd(&h[f32_key(f) >> 21], 1u);
    }
    if (nan) latch_error(p.err, LKV_ERR_NUMERIC, ci.head);
    __syncthreads();
    uint32_t* gh = p.hist + (size_t)ci.head * 2048;
    for (int i = threadIdx.x; i < 2048; i += kSelThreads)
        if (h[i]) atomicAdd(&gh[i], h[i]);
}

// ---- S2 --------------------------------------------------------------------------
// Find the bin holding the rank-`want` largest key of a histogram with `nbins`
// bins (bin value increasing with key).  Returns bin and the count above it.
template <int NT>
__device__ void find_bin_from_top(const uint32_t* cnt /*smem*/, int nbins, uint32_t want, uint32_t* s_scan,
                                  uint32_t* out_bin, uint32_t* out_above) {
    // exclusive scan in reverse bin order: above(bin) = sum of bins > bin
    const int per = (nbins + NT - 1) / NT;
    uint32_t local = 0;
    for (int q = 0; q < per; ++q) {
        const int r = threadIdx.x * per + q;  // reverse index
        if (r < nbins) local += cnt[nbins - 1 - r];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<NT>(local, s_scan, &tot);
    for (int q = 0; q < per; ++q) {
        const int r = threadIdx.x * per + q;
        if (r < nbins) {
            const uint32_t c = cnt[nbins - 1 - r];
            if (c && run < want && want <= run + c) {
                *out_bin = nbins - 1 - r;
                *out_above = run;
            }
            run += c;
        }
    }
    __syncthreads();
}

// ---- S2-S4 fused: one thread-block cluster per head ----------------------------------------------
// A head's chunks are split over the `cs` CTAs of a cluster (contiguous chunk ranges) while the
// grid still fits the resident slots, so a handful of heads (one rank's share of a head-sharded
// run) still use every SM; a few hundred heads run one CTA each.  Per CTA:
//   S2  the bin holding the b-th largest key, from the histogram K1 (or S1) built (every CTA of
//       the cluster derives the same bin).
//   S3  one pass over its chunks' scores in the float domain (the next step's loads in flight while
//       a step is processed): rows above the bin counted per chunk (one warp reduction per chunk),
//       rows inside it appended (position + key, warp-aggregated slots) and histogrammed on the
//       next 11 key bits on the spot.
//   S4  the cluster's histograms summed over distributed shared memory -> T's second digit; one
//       sweep over the candidates: digit above it -> above T (per-chunk counts), equal -> the last
//       10-bit histogram and a short list -> exact threshold key T and the number of T-equal rows
//       still needed; the short list settles the per-chunk counts.  Per-chunk output offsets: a
//       local chunk scan plus the cluster prefix of the lower ranks' totals (DSMEM).
// No global round trip between the phases and no inter-CTA spin (cluster barriers only).
constexpr int kPlanThreads = 512;
constexpr int kPlanBatch = 2;                     // chunks per step (one per half of the CTA)
constexpr int kPlanRows = kChunk * kPlanBatch / kPlanThreads;  // 16 contiguous rows of a chunk per thread
constexpr int kCandCap = 8192;                    // candidates per CTA in shared memory (rest: global)
constexpr int kPlanMaxCs = 8;                     // portable cluster size
constexpr int kPlanList = 512;                    // candidates sharing T's second digit (else a re-sweep)
constexpr size_t kPlanSmem = 2 * sizeof(uint32_t) * kCandCap;  // dynamic: positions + keys

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_ld_u32(const uint32_t* local, uint32_t rank) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsmem_map(smem_u32(local), rank)) : "memory");
    return v;
}

// cluster barrier; a plain CTA barrier when the cluster is this CTA alone (no cluster-scope fences)
__device__ __forceinline__ void plan_sync(uint32_t cs) {
    if (cs == 1) __syncthreads();
    else cluster_sync_all();
}

// sum the cluster's `nbins`-bin histograms `mine` (every rank's copy) into `out` (local)
__device__ __forceinline__ void cluster_hist_sum(const uint32_t* mine, uint32_t* out, int nbins, uint32_t cs) {
    plan_sync(cs);  // every rank's histogram complete
    if (cs == 1) {
        for (int i = threadIdx.x; i < nbins; i += kPlanThreads) out[i] = mine[i];
    } else {
        for (int i = threadIdx.x; i < nbins; i += kPlanThreads) {
            uint32_t v = 0;
            for (uint32_t r = 0; r < cs; ++r) v += dsmem_ld_u32(mine + i, r);
            out[i] = v;
        }
    }
    plan_sync(cs);  // every rank done reading `mine` (it is reused next)
}

__global__ void __launch_bounds__(kPlanThreads, 2) select_plan_kernel(const __grid_constant__ SelectParams p) {
    pdl_wait();
    __shared__ uint32_t cnt[2048];   // local histogram (read by the cluster)
    __shared__ uint32_t cnt2[2048];  // the cluster's sum
    __shared__ uint32_t c_gt[kMaxChunksPerHead];
    __shared__ uint32_t c_eq[kMaxChunksPerHead];
    extern __shared__ uint32_t plan_dyn[];
    uint32_t* s_cpos = plan_dyn;
    uint32_t* s_ckey = plan_dyn + kCandCap;
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_bin, s_above, s_ncand, s_nlist;
    __shared__ uint32_t s_lpos[kPlanList], s_lkey[kPlanList];  // candidates in T's 11-bit digit
    __shared__ uint32_t s_tot[2];    // this rank's equal-to-T and kept totals (read by higher ranks)
    const uint32_t cs = cluster_size(), crank = cluster_rank();
    const int head = blockIdx.x / cs;
    const int s_idx = head_seq(p.seq, head);
    const int t = p.seq.len[s_idx];
    const int b = p.budgets[head];
    HeadSel* st = p.state + head;
    if (b < 0 || b > t) {  // budget outside [0, t] (hard_topk, soft_topk.cpp:193); uniform over the cluster
        if (threadIdx.x == 0 && crank == 0) latch_error(p.err, LKV_ERR_BUDGET, head);
        return;
    }
    const int cph = (t + kChunk - 1) / kChunk;
    const int c_lo = (int)((int64_t)cph * crank / cs), c_hi = (int)((int64_t)cph * (crank + 1) / cs);
    const int nch = c_hi - c_lo;
    const int hs = head - s_idx * p.seq.n_layers * p.seq.n_kv_heads;
    const int cbase = p.chunk_base[s_idx] + hs * cph;
    const uint32_t mode = b == 0 ? kModeNone : (b == t ? kModeAll : kModeNormal);
    const int tid = threadIdx.x, lane = tid & 31;
    for (int c = tid; c < nch; c += kPlanThreads) {
        c_gt[c] = 0;
        c_eq[c] = 0;
    }
    if (tid == 0) s_ncand = 0;
    for (int i = tid; i < 2048; i += kPlanThreads) cnt[i] = 0;  // pass-A histogram, filled during S3
    uint32_t key_t = 0, need_eq = 0;
    if (mode == kModeNormal) {
        // S2
        const uint32_t* gh = p.hist + (size_t)head * 2048;
        {
            uint32_t hv[2048 / kPlanThreads];  // all loads in flight before the stores
#pragma unroll
            for (int q = 0; q < 2048 / kPlanThreads; ++q) hv[q] = gh[tid + q * kPlanThreads];
#pragma unroll
            for (int q = 0; q < 2048 / kPlanThreads; ++q) cnt2[tid + q * kPlanThreads] = hv[q];
        }
        __syncthreads();
        find_bin_from_top<kPlanThreads>(cnt2, 2048, (uint32_t)b, s_scan, &s_bin, &s_above);
        const uint32_t bin1 = s_bin;
        uint32_t rem = (uint32_t)b - s_above;
        // S3 in the float domain.  The bin's keys [bin1 << 21, ((bin1 + 1) << 21) - 1] are a float
        // interval, so a row lies above the bin iff x > g_thr and inside it iff x >= lo_f and not
        // above -- two compares per row, no key transform (IEEE compares treat -0.0 == +0.0, as the
        // key does; NaN was rejected by K1).
        const float* sc = p.scores + (size_t)head * p.seq.T;
        uint32_t* cand = p.cands + (size_t)head * p.seq.T + (size_t)c_lo * kChunk;  // overflow past kCandCap
        const uint32_t lo_key = bin1 << 21;
        const uint64_t hi1 = ((uint64_t)bin1 + 1) << 21;  // the first key above the bin
        const float lo_f = lo_key <= kKeyNegInf ? -INFINITY : key_to_f32(lo_key);
        const float g_thr = hi1 > kKeyPosInf ? INFINITY : float_below(key_to_f32((uint32_t)hi1));
        const int T = p.seq.T;
        const int full = t / kChunk;  // chunks whose 4096 rows are all inside the head
        // 16-byte loads when every head's scores are 16-byte aligned: branch-free (the address
        // clamped into the head's row stride) so a batch's loads are all issued before the first use
        const bool vec = ((reinterpret_cast<uintptr_t>(sc)) & 15) == 0 && (T & 3) == 0;
        // the loads of step i + 1 are issued before step i is processed (two register buffers)
        // a step covers kPlanBatch chunks, the CTA's halves one chunk each: thread tid reads rows
        // [j0, j0 + 16) of chunk c0 + u (u = tid / 256), four 16-byte loads
        const int u = tid / (kChunk / kPlanRows), j0 = (tid % (kChunk / kPlanRows)) * kPlanRows;
        auto load = [&](float (&v)[kPlanRows], int c0) {
            if (c0 + u >= c_hi) return;  // warp-uniform; process() skips it too
            if (vec) {
#pragma unroll
                for (int h = 0; h < kPlanRows / 4; ++h) {
                    const int r = min((c0 + u) * kChunk + j0 + 4 * h, T - 4);
                    const float4 f = __ldg(reinterpret_cast<const float4*>(sc + r));
                    v[4 * h + 0] = f.x;
                    v[4 * h + 1] = f.y;
                    v[4 * h + 2] = f.z;
                    v[4 * h + 3] = f.w;
                }
            } else {
                const int r = (c0 + u) * kChunk + j0;
#pragma unroll
                for (int q = 0; q < kPlanRows; ++q) v[q] = r + q < t ? __ldg(sc + r + q) : -INFINITY;
            }
        };
        // rows above the bin counted per chunk (one warp reduction); rows inside it appended
        // (warp-aggregated slots) with their key, and counted in the pass-A histogram
        auto process = [&](const float (&v)[kPlanRows], int c0) {
            {
                const int c = c0 + u;  // warp-uniform
                if (c >= c_hi) return;
                const int r0 = c * kChunk + j0;
                uint32_t gt = 0, cm = 0;  // rows above the bin; bit mask of the rows inside it
                if (c < full) {
#pragma unroll
                    for (int q = 0; q < kPlanRows; ++q) {
                        const bool above = v[q] > g_thr;
                        gt += above;
                        cm |= uint32_t(!above && v[q] >= lo_f) << q;
                    }
                } else {  // the head's last, partial chunk
#pragma unroll
                    for (int q = 0; q < kPlanRows; ++q) {
                        const bool ok = r0 + q < t;
                        const bool above = ok && v[q] > g_thr;
                        gt += above;
                        cm |= uint32_t(ok && !above && v[q] >= lo_f) << q;
                    }
                }
                const uint32_t wgt = __reduce_add_sync(0xffffffffu, gt);
                if (lane == 0 && wgt) atomicAdd(&c_gt[c - c_lo], wgt);
                if (!__any_sync(0xffffffffu, cm)) return;
                const uint32_t nc = __popc(cm);
                uint32_t incl = nc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                uint32_t base = 0;
                if (lane == 31) base = atomicAdd(&s_ncand, incl);
                base = __shfl_sync(0xffffffffu, base, 31) + incl - nc;
                while (cm) {  // only the rows inside the bin (a few % of them)
                    const int q = __ffs(cm) - 1;
                    cm &= cm - 1;
                    // v[q] by a 4-level select tree on the bits of q (registers cannot be indexed;
                    // re-reading the row from memory stalls on L2 when L1 has evicted the line)
                    float h8[8], h4[4], h2[2];
#pragma unroll
                    for (int z = 0; z < 8; ++z) h8[z] = (q & 8) ? v[z + 8] : v[z];
#pragma unroll
                    for (int z = 0; z < 4; ++z) h4[z] = (q & 4) ? h8[z + 4] : h8[z];
#pragma unroll
                    for (int z = 0; z < 2; ++z) h2[z] = (q & 2) ? h4[z + 2] : h4[z];
                    const uint32_t key = f32_key((q & 1) ? h2[1] : h2[0]);
                    atomicAdd(&cnt[(key >> 10) & 2047u], 1u);  // S4 pass A, fused
                    if (base < kCandCap) {
                        s_cpos[base] = (uint32_t)(r0 + q);
                        s_ckey[base] = key;
                    } else {
                        cand[base - kCandCap] = (uint32_t)(r0 + q);
                    }
                    ++base;
                }
            }
        };
        {
            float va[kPlanRows], vb[kPlanRows];
            int c0 = c_lo;
            if (c0 < c_hi) load(va, c0);
            while (c0 < c_hi) {
                if (c0 + kPlanBatch < c_hi) load(vb, c0 + kPlanBatch);
                process(va, c0);
                c0 += kPlanBatch;
                if (c0 >= c_hi) break;
                if (c0 + kPlanBatch < c_hi) load(va, c0 + kPlanBatch);
                process(vb, c0);
                c0 += kPlanBatch;
            }
        }
        __syncthreads();
        const uint32_t n_cand = s_ncand;
        auto cand_key = [&](uint32_t i) -> uint32_t {
            return i < kCandCap ? s_ckey[i] : f32_key(sc[cand[i - kCandCap]]);
        };
        // S4 pass A (histogram of key bits [10, 21) built during S3): the digit of T
        cluster_hist_sum(cnt, cnt2, 2048, cs);
        find_bin_from_top<kPlanThreads>(cnt2, 2048, rem, s_scan, &s_bin, &s_above);
        const uint32_t binA = s_bin;
        rem -= s_above;
        // pass B, one sweep over the candidates: digit above binA -> above T, counted per chunk (one
        // atomic per (warp, chunk)); digit == binA -> low-10-bit histogram and the short list of
        // rows whose order against T is still open
        for (int i = tid; i < 1024; i += kPlanThreads) cnt[i] = 0;
        if (tid == 0) s_nlist = 0;
        __syncthreads();
        for (uint32_t i0 = 0; i0 < n_cand; i0 += kPlanThreads) {
            const uint32_t i = i0 + tid;
            bool above = false;
            uint32_t ch = 0;
            if (i < n_cand) {
                const uint32_t pos = i < kCandCap ? s_cpos[i] : cand[i - kCandCap];
                const uint32_t kk = cand_key(i);
                const uint32_t d = (kk >> 10) & 2047u;
                ch = pos / kChunk - c_lo;
                above = d > binA;
                if (d == binA) {
                    atomicAdd(&cnt[kk & 1023u], 1u);
                    const uint32_t j = atomicAdd(&s_nlist, 1u);
                    if (j < kPlanList) {
                        s_lpos[j] = pos;
                        s_lkey[j] = kk;
                    }
                }
            }
            // the list is in append order, mostly one chunk per warp: one atomic when all lanes
            // agree, else one per lane
            const uint32_t ch0 = __shfl_sync(0xffffffffu, ch, 0);
            if (__all_sync(0xffffffffu, ch == ch0)) {
                const uint32_t na = __popc(__ballot_sync(0xffffffffu, above));
                if (lane == 0 && na) atomicAdd(&c_gt[ch0], na);
            } else if (above) {
                atomicAdd(&c_gt[ch], 1u);
            }
        }
        cluster_hist_sum(cnt, cnt2, 1024, cs);
        find_bin_from_top<kPlanThreads>(cnt2, 1024, rem, s_scan, &s_bin, &s_above);
        key_t = (bin1 << 21) | (binA << 10) | s_bin;
        need_eq = rem - s_above;
        // the open rows: above T or equal to T, per chunk (the list, or -- when it overflowed -- the
        // candidates again)
        const uint32_t n_list = s_nlist;
        const bool listed = n_list <= (uint32_t)kPlanList;
        const uint32_t n_open = listed ? n_list : n_cand;
        for (uint32_t i = tid; i < n_open; i += kPlanThreads) {
            uint32_t pos, kk;
            if (listed) {
                pos = s_lpos[i];
                kk = s_lkey[i];
            } else {
                pos = i < kCandCap ? s_cpos[i] : cand[i - kCandCap];
                kk = cand_key(i);
                if (((kk >> 10) & 2047u) != binA) continue;
            }
            const uint32_t ch = pos / kChunk - c_lo;
            if (kk > key_t) atomicAdd(&c_gt[ch], 1u);
            else if (kk == key_t) atomicAdd(&c_eq[ch], 1u);
        }
    }
    __syncthreads();
    // chunk scan over this rank's chunks (eq_before and out_base in index order), offset by the
    // lower ranks' totals
    constexpr int kPer = kMaxChunksPerHead / kPlanThreads;
    uint32_t gtv[kPer], eqv[kPer], eq_loc = 0;
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
        const int c = tid * kPer + h;
        gtv[h] = eqv[h] = 0;
        if (c < nch) {
            if (mode == kModeAll) gtv[h] = (uint32_t)min(kChunk, t - (c_lo + c) * kChunk);
            else if (mode == kModeNormal) gtv[h] = c_gt[c];
            eqv[h] = c_eq[c];
        }
        eq_loc += eqv[h];
    }
    uint32_t eq_tot;
    uint32_t eqb = block_exclusive_scan<kPlanThreads>(eq_loc, s_scan, &eq_tot);
    if (tid == 0) s_tot[0] = eq_tot;
    plan_sync(cs);
    uint32_t eq_base = 0;
    for (uint32_t r = 0; r < crank; ++r) eq_base += dsmem_ld_u32(&s_tot[0], r);
    eqb += eq_base;
    uint32_t keptv[kPer], eqbv[kPer], kept_loc = 0;
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
        eqbv[h] = eqb;
        const uint32_t take = need_eq > eqb ? min(need_eq - eqb, eqv[h]) : 0u;
        keptv[h] = gtv[h] + take;
        kept_loc += keptv[h];
        eqb += eqv[h];
    }
    uint32_t kept_tot;
    uint32_t ob = block_exclusive_scan<kPlanThreads>(kept_loc, s_scan, &kept_tot);
    if (tid == 0) s_tot[1] = kept_tot;
    plan_sync(cs);
    uint32_t out_base = 0;
    for (uint32_t r = 0; r < crank; ++r) out_base += dsmem_ld_u32(&s_tot[1], r);
    ob += out_base;
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
        const int c = tid * kPer + h;
        if (c < nch) {
            p.chunk_out[cbase + c_lo + c] = ob;
            p.chunk_eqb[cbase + c_lo + c] = eqbv[h];
        }
        ob += keptv[h];
    }
    if (tid == 0 && crank == cs - 1) {
        st->mode = mode;
        st->key_t = key_t;
        st->need_eq = need_eq;
        p.out_lens[head] = b;
        if (out_base + kept_tot != (uint32_t)b) latch_error(p.err, LKV_ERR_NUMERIC, head);  // internal consistency
    }
    if (cs > 1) cluster_sync_all();  // no rank exits while another may still read its shared memory
}

// ---- row gather (16-byte vectors) ----------------------------------------------------------
constexpr int kGatherUnroll = 8;  // 16-byte loads in flight per thread and tensor
// 2^log2_units 16-byte vectors per row (head_dim * elem / 16); lanes walk (row, vector)
// pairs so a warp moves whole rows with coalesced 16-byte accesses.
// K and V rows of the same kept positions in one loop: twice the loads in flight per thread
__device__ __forceinline__ void gather_rows_kv(const uint4* __restrict__ ks, const uint4* __restrict__ vs,
                                               uint4* __restrict__ kd, uint4* __restrict__ vd,
                                               const int32_t* rows /*smem*/, int n_rows, int log2_units, int tid,
                                               int nthreads) {
    const int units = 1 << log2_units;
    const int total = n_rows << log2_units;
    int u = tid;
    constexpr int U = kGatherUnroll;
    for (; u + (U - 1) * nthreads < total; u += U * nthreads) {
        uint4 a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int uu = u + k * nthreads;
            const size_t off = ((size_t)rows[uu >> log2_units] << log2_units) + (uu & (units - 1));
            a[k] = __ldg(ks + off);
            b[k] = __ldg(vs + off);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            __stcs(kd + u + k * nthreads, a[k]);
            __stcs(vd + u + k * nthreads, b[k]);
        }
    }
    for (; u < total; u += nthreads) {
        const size_t off = ((size_t)rows[u >> log2_units] << log2_units) + (u & (units - 1));
        __stcs(kd + u, __ldg(ks + off));
        __stcs(vd + u, __ldg(vs + off));
    }
}

// ---- S5 --------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelThreads) select_emit_kernel(const __grid_constant__ SelectParams p) {
    pdl_wait();
    __shared__ int32_t s_pos[kChunk];
    __shared__ uint32_t s_scan[kSelThreads / 32 + 1];
    const ChunkInfo ci = decode_chunk(p, blockIdx.x);
    const int b = p.budgets[ci.head];
    if (b < 0 || b > ci.t) return;
    const HeadSel* st = p.state + ci.head;
    const uint32_t mode = st->mode;
    if (mode == kModeNone) return;
    const uint32_t key_t = st->key_t, need_eq = st->need_eq;
    const uint32_t out_base = p.chunk_out[blockIdx.x];
    const uint32_t eqb = p.chunk_eqb[blockIdx.x];
    const float* sc = p.scores + (size_t)ci.head * p.seq.T + ci.c0;

    const int j0 = threadIdx.x * kPerThread;
    uint32_t keys[kPerThread];
    uint32_t n_eq = 0;
    load_keys16(sc, j0, ci.n, keys);
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) n_eq += (j0 + q < ci.n) && keys[q] == key_t;
    uint32_t tot;
    uint32_t eq_rank = eqb + block_exclusive_scan<kSelThreads>(n_eq, s_scan, &tot);
    uint32_t keepmask = 0, n_keep = 0;
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
        const int j = j0 + q;
        bool keep = false;
        if (j < ci.n) {
            if (mode == kModeAll) keep = true;
            else if (keys[q] > key_t) keep = true;
            else if (keys[q] == key_t) {
                keep = eq_rank < need_eq;
                ++eq_rank;
            }
        }
        keepmask |= uint32_t(keep) << q;
        n_keep += keep;
    }
    uint32_t slot = block_exclusive_scan<kSelThreads>(n_keep, s_scan, &tot);
    const int64_t obase = p.offsets[ci.head] + out_base;
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
        if (keepmask >> q & 1u) {
            const int32_t pos = ci.c0 + j0 + q;
            p.out_pos[obase + slot] = pos;
            s_pos[slot] = pos;
            ++slot;
        }
    }
    if (!p.gather) return;
    __syncthreads();
    const int lu = 31 - __clz(p.row_bytes / 16);
    const size_t head_row0 = (size_t)ci.head * p.seq.T;
    gather_rows_kv(static_cast<const uint4*>(p.keys) + (head_row0 << lu),
                   static_cast<const uint4*>(p.values) + (head_row0 << lu), static_cast<uint4*>(p.out_keys) + (obase << lu),
                   static_cast<uint4*>(p.out_values) + (obase << lu), s_pos, (int)tot, lu, threadIdx.x, kSelThreads);
}

// ---- standalone compaction: positions given (cache_from_trace, model.cpp:289-315) -------------

constexpr int kCompactRows = 256;

// A position outside [0, t) (or a head whose rows overrun its capacity) is a contract_error, as
// the reference's bounds checks raise (model.cpp:298-312, evictsim.cpp:104-109): it is latched in
// the caller's workspace and the offending rows are not written (never silently replaced).
__global__ void __launch_bounds__(256) compact_kernel(const __grid_constant__ CompactParams p) {
    __shared__ int32_t s_pos[kCompactRows];
    __shared__ int s_bad;
    const int head = blockIdx.y;
    const int r0 = blockIdx.x * kCompactRows;
    const int len = p.lens[head];
    if (r0 >= len) return;
    const int n = min(kCompactRows, len - r0);
    const int t = p.seq.len[head_seq(p.seq, head)];
    const int64_t obase = p.offsets[head] + r0;
    if (len < 0 || p.offsets[head] + len > p.offsets[head + 1]) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_CONTRACT, head);
        return;
    }
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += 256) {
        const int32_t pos = p.positions[obase + i];
        if (pos < 0 || pos >= t) s_bad = 1;
        s_pos[i] = pos;
    }
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) latch_error(p.err, LKV_ERR_CONTRACT, head);
        return;
    }
    const int lu = 31 - __clz(p.row_bytes / 16);
    const size_t head_row0 = (size_t)head * p.seq.T;
    gather_rows_kv(static_cast<const uint4*>(p.keys) + (head_row0 << lu),
                   static_cast<const uint4*>(p.values) + (head_row0 << lu), static_cast<uint4*>(p.out_keys) + (obase << lu),
                   static_cast<uint4*>(p.out_values) + (obase << lu), s_pos, n, lu, threadIdx.x, 256);
}

// ---- cache_from_trace on the device: compaction by a mask scan (model.cpp:289-315) -------------
// Row j of head i is kept iff masks[i * mask_ld + j] != 0 (j < t), ascending.  Three passes over
// 4096-row chunks: count, per-head chunk scan (-> lens), emit (positions + 16-byte row gather).
__device__ __forceinline__ ChunkInfo trace_chunk(const TraceParams& p, int chunk) {
    int s = 0;
    while (s + 1 < p.seq.n_seq && p.chunk_base[s + 1] <= chunk) ++s;
    const int t = p.seq.len[s];
    const int cph = (t + kChunk - 1) / kChunk;
    const int local = chunk - p.chunk_base[s];
    const int hs = local / cph;
    ChunkInfo ci;
    ci.c = local - hs * cph;
    ci.head = s * p.seq.n_layers * p.seq.n_kv_heads + hs;
    ci.cbase = chunk - ci.c;
    ci.t = t;
    ci.c0 = ci.c * kChunk;
    ci.n = min(kChunk, t - ci.c0);
    return ci;
}

__device__ __forceinline__ uint32_t trace_keep16(const TraceParams& p, const ChunkInfo& ci, int j0) {
    const int32_t* m = p.masks + (size_t)ci.head * p.mask_ld + ci.c0;
    uint32_t keep = 0;
    if (j0 + kPerThread <= ci.n && (reinterpret_cast<uintptr_t>(m + j0) & 15) == 0) {
        const int4* v = reinterpret_cast<const int4*>(m + j0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int4 x = __ldg(v + q);
            keep |= uint32_t(x.x != 0) << (4 * q) | uint32_t(x.y != 0) << (4 * q + 1) |
                    uint32_t(x.z != 0) << (4 * q + 2) | uint32_t(x.w != 0) << (4 * q + 3);
        }
    } else {
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) keep |= uint32_t(j0 + q < ci.n && __ldg(m + j0 + q) != 0) << q;
    }
    return keep;
}

__global__ void __launch_bounds__(kSelThreads) trace_count_kernel(const __grid_constant__ TraceParams p) {
    __shared__ uint32_t s_scan[kSelThreads / 32 + 1];
    const ChunkInfo ci = trace_chunk(p, blockIdx.x);
    const uint32_t n = __popc(trace_keep16(p, ci, threadIdx.x * kPerThread));
    uint32_t tot;
    block_exclusive_scan<kSelThreads>(n, s_scan, &tot);
    if (threadIdx.x == 0) p.chunk_cnt[blockIdx.x] = tot;
}

// one CTA per head: chunk counts -> exclusive chunk bases (in place), head total -> counts
__global__ void __launch_bounds__(kSelThreads) trace_scan_kernel(const __grid_constant__ TraceParams p) {
    __shared__ uint32_t s_scan[kSelThreads / 32 + 1];
    const int head = blockIdx.x;
    const int s_idx = head_seq(p.seq, head);
    const int t = p.seq.len[s_idx];
    const int cph = (t + kChunk - 1) / kChunk;
    const int hs = head - s_idx * p.seq.n_layers * p.seq.n_kv_heads;
    uint32_t* cc = p.chunk_cnt + p.chunk_base[s_idx] + hs * cph;
    constexpr int kPer = kMaxChunksPerHead / kSelThreads;
    uint32_t v[kPer], local = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int c = threadIdx.x * kPer + q;
        v[q] = c < cph ? cc[c] : 0u;
        local += v[q];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<kSelThreads>(local, s_scan, &tot);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int c = threadIdx.x * kPer + q;
        if (c < cph) cc[c] = run;
        run += v[q];
    }
    if (threadIdx.x == 0) p.counts[head] = (int32_t)tot;
}

__global__ void __launch_bounds__(kSelThreads) trace_emit_kernel(const __grid_constant__ TraceParams p) {
    __shared__ int32_t s_pos[kChunk];
    __shared__ uint32_t s_scan[kSelThreads / 32 + 1];
    const ChunkInfo ci = trace_chunk(p, blockIdx.x);
    const int64_t o0 = p.offsets[ci.head], o1 = p.offsets[ci.head + 1];
    const int32_t len = p.counts[ci.head];
    if (o0 < 0 || o0 + len > o1 || o1 > p.capacity) {  // the ragged cache cannot hold this head
        if (threadIdx.x == 0 && ci.c == 0) latch_error(p.err, LKV_ERR_CONTRACT, ci.head);
        return;
    }
    const int j0 = threadIdx.x * kPerThread;
    const uint32_t keep = trace_keep16(p, ci, j0);
    uint32_t tot;
    uint32_t slot = block_exclusive_scan<kSelThreads>(__popc(keep), s_scan, &tot);
    const int64_t obase = o0 + p.chunk_cnt[blockIdx.x];
    uint32_t k = keep;
    while (k) {
        const int q = __ffs(k) - 1;
        k &= k - 1;
        const int32_t pos = ci.c0 + j0 + q;
        p.out_pos[obase + slot] = pos;
        s_pos[slot] = pos;
        ++slot;
    }
    if (!p.gather || tot == 0) return;
    __syncthreads();
    const int lu = 31 - __clz(p.row_bytes / 16);
    const size_t head_row0 = (size_t)ci.head * p.seq.T;
    gather_rows_kv(static_cast<const uint4*>(p.keys) + (head_row0 << lu),
                   static_cast<const uint4*>(p.values) + (head_row0 << lu), static_cast<uint4*>(p.out_keys) + (obase << lu),
                   static_cast<uint4*>(p.out_values) + (obase << lu), s_pos, (int)tot, lu, threadIdx.x, kSelThreads);
}

static int trace_total_chunks(TraceParams& p) {
    int64_t acc = 0;
    for (int s = 0; s < p.seq.n_seq; ++s) {
        p.chunk_base[s] = (int32_t)acc;
        acc += (int64_t)p.seq.n_layers * p.seq.n_kv_heads * ((p.seq.len[s] + kChunk - 1) / kChunk);
    }
    p.chunk_base[p.seq.n_seq] = (int32_t)acc;
    return (int)acc;
}

cudaError_t launch_trace_counts(TraceParams p, int n_heads, cudaStream_t stream) {
    const int chunks = trace_total_chunks(p);
    if (chunks == 0) return cudaSuccess;
    trace_count_kernel<<<chunks, kSelThreads, 0, stream>>>(p);
    trace_scan_kernel<<<n_heads, kSelThreads, 0, stream>>>(p);
    note_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_trace_emit(TraceParams p, cudaStream_t stream) {
    const int chunks = trace_total_chunks(p);
    if (chunks == 0) return cudaSuccess;
    trace_emit_kernel<<<chunks, kSelThreads, 0, stream>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

// ---- host launchers --------------------------------------------------------------------------
int select_total_chunks(SelectParams& p) {
    int64_t acc = 0;
    for (int s = 0; s < p.seq.n_seq; ++s) {
        p.chunk_base[s] = (int32_t)acc;
        acc += (int64_t)p.seq.n_layers * p.seq.n_kv_heads * ((p.seq.len[s] + kChunk - 1) / kChunk);
    }
    p.chunk_base[p.seq.n_seq] = (int32_t)acc;
    return (int)acc;
}

cudaError_t launch_select(SelectParams p, int n_heads, cudaStream_t stream) {
    const int chunks = select_total_chunks(p);
    if (chunks == 0) return cudaSuccess;
    if (!p.hist_ready) {
        const cudaError_t e = cudaMemsetAsync(p.hist, 0, sizeof(uint32_t) * 2048 * (size_t)n_heads, stream);
        if (e != cudaSuccess) return e;
        select_hist_kernel<<<chunks, kSelThreads, 0, stream>>>(p);
        note_launches(1);
    }
    cudaError_t e;
    const cudaError_t attr =
        cudaFuncSetAttribute(select_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlanSmem);
    if (attr != cudaSuccess) return attr;
    // cluster size: split heads while the grid still fits the resident slots (2 CTAs / SM), never
    // below one chunk per CTA (cs <= the longest head's chunk count), at most the portable 8
    int dev = 0, sms = 148, max_cph = 1;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int s = 0; s < p.seq.n_seq; ++s) max_cph = max(max_cph, (p.seq.len[s] + kChunk - 1) / kChunk);
    int cs = 1;
    while (cs < kPlanMaxCs && 2 * cs <= max_cph && (int64_t)n_heads * cs * 2 <= 2 * (int64_t)sms) cs *= 2;
    if ((e = launch_pdl_cluster(select_plan_kernel, dim3(n_heads * cs), dim3(kPlanThreads), kPlanSmem, stream, cs,
                                p)) != cudaSuccess)
        return e;
    if ((e = launch_pdl(select_emit_kernel, dim3(chunks), dim3(kSelThreads), 0, stream, p)) != cudaSuccess) return e;
    note_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_compact(const CompactParams& p, int n_heads, cudaStream_t stream) {
    int64_t maxt = 0;
    for (int s = 0; s < p.seq.n_seq; ++s) maxt = maxt > p.seq.len[s] ? maxt : p.seq.len[s];
    const int gx = (int)((maxt + kCompactRows - 1) / kCompactRows);
    if (gx == 0 || n_heads == 0) return cudaSuccess;
    compact_kernel<<<dim3(gx, n_heads), 256, 0, stream>>>(p);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace lkv_dev
