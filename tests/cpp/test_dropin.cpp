// C++ drop-in tests: the reference's own hot-path test expectations (proj/tests/*.cpp)
// exercised through lkv::b200:: (include/lkv_b200_dropin.hpp) on the B200.
// Built by `make -C paper_2605_06676_b200 test_dropin`; run by tests/test_dropin_cpp.py.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../include/lkv_b200_dropin.hpp"

using namespace lkv::b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                 \
    do {                                                                         \
        bool ok_ = false;                                                        \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const T&) {                                                     \
            ok_ = true;                                                          \
        } catch (...) {                                                          \
        }                                                                        \
        CHECK(ok_);                                                              \
    } while (0)

static std::vector<double> uniform(size_t n, double lo, double hi, unsigned seed) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> u(lo, hi);
    std::vector<double> v(n);
    for (double& x : v) x = u(g);
    return v;
}

static double f32(double x) { return (double)(float)x; }

// round to bf16 (nearest even), as the device sees bf16 inputs
static double bf16(double x) {
    float f = (float)x;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
    std::memcpy(&f, &u, 4);
    return (double)f;
}

static Mlp2 make_mlp(int in, int hidden, unsigned seed) {
    Mlp2 m;
    m.in = in;
    m.hidden = hidden;
    m.w1 = uniform((size_t)in * hidden, -1.0 / std::sqrt(in), 1.0 / std::sqrt(in), seed);
    m.b1.assign((size_t)hidden, 0.0);  // init_mlp2: b1 = 0 (policy.cpp:18-28)
    m.w2 = uniform((size_t)hidden, -0.5, 0.5, seed + 1);
    return m;
}

static void test_budgets() {
    // test_policy.cpp:51-60 equal scores allocate the target ratio everywhere
    std::vector<double> eq(8, 0.3);
    BudgetTable t = allocate_budgets(eq, 0.15, 4, 2);
    double sum = 0.0;
    for (double r : t.ratios) {
        CHECK(std::fabs(r - 0.15) <= 1e-12 * 0.15);
        sum += r;
    }
    CHECK(std::fabs(sum - 1.2) <= 1e-12 * 1.2);
    // :62-68 a dominant head receives the strictly greatest ratio
    std::vector<double> dom{0, 0, 5.0, 0, 0, 0, 0, 0};
    BudgetTable d = allocate_budgets(dom, 0.15, 4, 2);
    for (int i = 0; i < 8; ++i)
        if (i != 2) CHECK(d.ratios[2] > d.ratios[(size_t)i]);
    // :107-116 floor fixture on a hand-built table
    BudgetTable f;
    f.n_layers = 1;
    f.n_kv_heads = 3;
    f.target_ratio = 0.15;
    f.ratios = {0.15, 0.15, 0.003};
    CHECK((freeze_budgets(f, 1000) == std::vector<int>{150, 150, 3}));
    CHECK((freeze_budgets(f, 200000) == std::vector<int>{30000, 30000, 600}));
    CHECK((freeze_budgets(f, 100) == std::vector<int>{15, 15, 0}));
    CHECK_THROWS_AS(freeze_budgets(f, 0), contract_error);
    // domain errors (policy.cpp:111-113)
    CHECK_THROWS_AS(allocate_budgets(eq, 0.0, 4, 2), budget_error);
    CHECK_THROWS_AS(allocate_budgets(eq, 1.0, 4, 2), budget_error);
    CHECK_THROWS_AS(allocate_budgets(eq, 0.2, 4, 3), contract_error);
    std::vector<double> bad{0.0, NAN, 1.0};
    CHECK_THROWS_AS(allocate_budgets(bad, 0.3, 1, 3), numeric_error);
    std::vector<double> huge{0.0, 1e301, 1.0};
    CHECK_THROWS_AS(allocate_budgets(huge, 0.3, 1, 3), overflow_guard_error);
    // exact-sum freezing hits the total
    auto logits = uniform(256, -2.0, 2.0, 7);
    BudgetTable big = allocate_budgets(logits, 0.15, 32, 8);
    auto ex = freeze_budgets_exact(big, 32768);
    long long s = 0;
    for (int b : ex) s += b;
    CHECK(s == 1258291);
}

static void test_budget_csv() {  // policy.cpp:301-311
    std::vector<double> eq(4, 0.3);
    BudgetTable t = allocate_budgets(eq, 0.15, 2, 2);
    CHECK(budget_table_csv(t) == "layer,head,ratio\n0,0,0.150000\n0,1,0.150000\n1,0,0.150000\n1,1,0.150000\n");
}

static void test_hard_topk() {  // test_soft_topk.cpp:190-199
    std::vector<float> x{0.1f, 0.9f, 0.5f};
    CHECK((hard_topk(x, 2) == std::vector<int>{0, 1, 1}));
    CHECK((hard_topk(x, 0) == std::vector<int>{0, 0, 0}));
    CHECK((hard_topk(x, 3) == std::vector<int>{1, 1, 1}));
    std::vector<float> ties{0.7f, 0.2f, 0.7f};
    CHECK((inference_select(ties, 1) == std::vector<int>{1, 0, 0}));
    CHECK_THROWS_AS(hard_topk(x, 4), budget_error);
    CHECK_THROWS_AS(hard_topk(x, -1), budget_error);
}

static void test_token_scores() {  // test_policy.cpp:118-139 on the desk geometry (d = 16, 2d -> d -> 1)
    const int t = 6, d = 16;
    Mlp2 m = make_mlp(2 * d, d, 13);
    auto k = uniform((size_t)t * d, -1, 1, 14), v = uniform((size_t)t * d, -1, 1, 15);
    for (int c = 0; c < d; ++c) {
        k[(size_t)4 * d + c] = k[(size_t)2 * d + c];
        v[(size_t)4 * d + c] = v[(size_t)2 * d + c];
    }
    auto u = token_scores(k, v, t, d, m);
    CHECK(u[2] == u[4]);
    std::vector<double> z((size_t)t * d, 0.0);
    for (double s : token_scores(z, z, t, d, m)) CHECK(s == 0.0);
    // fp64 formula on the fp32-rounded inputs (policy.cpp:30-34): 1e-5 relative
    double worst = 0.0, scale = 0.0;
    for (int r = 0; r < t; ++r) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) {
            double h = m.b1[(size_t)j];
            for (int i = 0; i < d; ++i) h += f32(k[(size_t)r * d + i]) * f32(m.w1[(size_t)i * d + j]);
            for (int i = 0; i < d; ++i) h += f32(v[(size_t)r * d + i]) * f32(m.w1[(size_t)(d + i) * d + j]);
            s += h / (1.0 + std::exp(-h)) * f32(m.w2[(size_t)j]);
        }
        worst = std::fmax(worst, std::fabs(s - u[(size_t)r]));
        scale = std::fmax(scale, std::fabs(s));
    }
    CHECK(worst / (scale + 1e-12) <= 1e-5);
    CHECK_THROWS_AS(token_scores(k, std::vector<double>(3), t, d, m), contract_error);
}

static KvTrace make_trace(int L, int H, int d, int t, unsigned seed) {
    KvTrace tr;
    tr.n_layers = L;
    tr.n_kv_heads = H;
    tr.head_dim = d;
    tr.t = t;
    for (int h = 0; h < L * H; ++h) {
        tr.keys.push_back(uniform((size_t)t * d, -1, 1, seed + 2 * h));
        tr.values.push_back(uniform((size_t)t * d, -1, 1, seed + 2 * h + 1));
    }
    return tr;
}

static void test_cache_and_prefill() {
    const int L = 2, H = 2, d = 16, t = 24;
    KvTrace tr = make_trace(L, H, d, t, 100);
    // cache_from_trace (model.cpp:289-315)
    std::vector<std::vector<int>> masks((size_t)L * H, std::vector<int>((size_t)t, 0));
    std::mt19937 g(42);
    for (auto& m : masks) {
        for (int j = 0; j < t; ++j) m[(size_t)j] = (g() % 10) < 6;
        m[0] = 1;
    }
    KvCache c = cache_from_trace(tr, masks);
    for (int h = 0; h < L * H; ++h) {
        const HeadCache& hc = c.heads[(size_t)h];
        int r = 0;
        for (int j = 0; j < t; ++j) {
            if (!masks[(size_t)h][(size_t)j]) continue;
            CHECK(hc.retained_positions[(size_t)r] == j);
            for (int q = 0; q < d; ++q) CHECK(hc.keys[(size_t)r * d + q] == f32(tr.keys[(size_t)h][(size_t)j * d + q]));
            ++r;
        }
        CHECK(hc.retained() == r);
    }
    // test_evictsim.cpp:82-101 full budgets keep every row
    std::vector<Mlp2> scorers;
    for (int h = 0; h < L * H; ++h) scorers.push_back(make_mlp(2 * d, d, 300 + h));
    auto [full, rep] = prefill_with_eviction(tr, std::vector<int>((size_t)L * H, t), scorers, Activation::silu);
    for (int h = 0; h < L * H; ++h) {
        CHECK(rep.retained_per_head[(size_t)h] == t);
        for (int j = 0; j < t * d; ++j) CHECK(full.heads[(size_t)h].keys[(size_t)j] == f32(tr.keys[(size_t)h][(size_t)j]));
    }
    // :134-141 budgets beyond the context length are rejected
    CHECK_THROWS_AS(prefill_with_eviction(tr, std::vector<int>((size_t)L * H, t + 1), scorers, Activation::silu),
                    budget_error);
    CHECK_THROWS_AS(prefill_with_eviction(tr, std::vector<int>(3, 1), scorers, Activation::silu), contract_error);
    // :143-160 retained counts equal the budgets, positions strictly increasing; and the kept rows are
    // the top-b of the device scores (ties -> lowest index)
    std::vector<int> budgets{5, 0, 24, 11};
    auto [cache, rep2] = prefill_with_eviction(tr, budgets, scorers, Activation::silu);
    for (int h = 0; h < L * H; ++h) {
        const auto& p = cache.heads[(size_t)h].retained_positions;
        CHECK((int)p.size() == budgets[(size_t)h]);
        for (size_t i = 1; i < p.size(); ++i) CHECK(p[i] > p[i - 1]);
        auto u = token_scores(tr.keys[(size_t)h], tr.values[(size_t)h], t, d, scorers[(size_t)h]);
        std::vector<float> uf(u.begin(), u.end());
        auto mask = inference_select(uf, budgets[(size_t)h]);
        std::vector<int> want;
        for (int j = 0; j < t; ++j)
            if (mask[(size_t)j]) want.push_back(j);
        CHECK(want == p);
    }
    CHECK(rep2.scoring_ops == (int64_t)L * H * t * (2 * d * d + 3 * d));  // evictsim.cpp:172
}

static void test_decode() {
    // decode equals the dense fp64 attention over the (fp32-stored) cache plus the new row;
    // a zero-budget head attends to the new token only (test_evictsim.cpp:119-132)
    const int L = 2, H = 2, d = 16, t = 40, Hq = 8, G = Hq / H;
    KvTrace tr = make_trace(L, H, d, t, 500);
    std::vector<std::vector<int>> masks((size_t)L * H, std::vector<int>((size_t)t, 1));
    masks[1].assign((size_t)t, 0);
    KvCache cache = cache_from_trace(tr, masks);
    for (int step = 0; step < 3; ++step) {
        auto q = uniform((size_t)L * Hq * d, -1, 1, 900 + step);
        auto kn = uniform((size_t)L * H * d, -1, 1, 910 + step);
        auto vn = uniform((size_t)L * H * d, -1, 1, 920 + step);
        KvCache before = cache;
        auto out = decode_attention(cache, q, Hq, kn, vn);
        CHECK(cache.tokens_seen == t + step + 1);
        double worst = 0.0, scale = 0.0;
        for (int l = 0; l < L; ++l)
            for (int qh = 0; qh < Hq; ++qh) {
                const int h = l * H + qh / G;
                std::vector<double> K = before.heads[(size_t)h].keys, V = before.heads[(size_t)h].values;
                for (int c = 0; c < d; ++c) {
                    K.push_back(kn[(size_t)h * d + c]);
                    V.push_back(vn[(size_t)h * d + c]);
                }
                const int n = (int)K.size() / d;
                std::vector<double> s((size_t)n);
                double mx = -INFINITY;
                for (int j = 0; j < n; ++j) {
                    double dot = 0.0;
                    for (int c = 0; c < d; ++c) dot += f32(q[((size_t)l * Hq + qh) * d + c]) * f32(K[(size_t)j * d + c]);
                    s[(size_t)j] = dot / std::sqrt((double)d);
                    mx = std::fmax(mx, s[(size_t)j]);
                }
                double z = 0.0;
                for (double& x : s) z += (x = std::exp(x - mx));
                for (int c = 0; c < d; ++c) {
                    double o = 0.0;
                    for (int j = 0; j < n; ++j) o += s[(size_t)j] / z * f32(V[(size_t)j * d + c]);
                    const double got = out[((size_t)l * Hq + qh) * d + c];
                    worst = std::fmax(worst, std::fabs(o - got));
                    scale = std::fmax(scale, std::fabs(o));
                    if (h == 1 && step == 0) CHECK(std::fabs(got - f32(vn[(size_t)h * d + c])) <= 1e-6);
                }
            }
        CHECK(worst / (scale + 1e-12) <= 1e-5);
    }
    CHECK(cache.heads[1].retained() == 3);
}

static void test_memory() {  // test_evictsim.cpp:45-80
    MemoryModel mm;
    CHECK(std::fabs(kv_memory_bytes(mm, 1.0).full_bytes - 26214400000.0) < 1.0);
    CHECK(std::fabs(kv_memory_bytes(mm, 0.15).reduction_factor - 6.67) < 0.01);
    CHECK_THROWS_AS(kv_memory_bytes(mm, 0.0), budget_error);
    CHECK_THROWS_AS(kv_memory_bytes(mm, 1.5), budget_error);
    MemoryModel s;
    s.n_layers = 1;
    s.n_kv_heads = 2;
    s.head_dim = 4;
    s.tokens = 100;
    MemoryReport r = kv_memory_bytes(s, std::vector<int>{15, 14});
    CHECK(r.full_bytes == 2 * 4 * 2.0 * 2 * 100);
    CHECK(r.compressed_bytes == (15 + 14) * 4 * 2.0 * 2);
}

static void test_checkpoint(const char* dir) {  // the reference's own lkv_params.bin (tests/golden)
    if (!dir) return;
    const std::string base(dir);
    LkvParams p = load_lkv_params(base + "/lkv_params_l2h4d128.bin");
    CHECK(p.n_layers == 2 && p.n_kv_heads == 4 && p.d_head == 128 && p.d_e == 32);
    CHECK(p.token_scorers.size() == 8);
    auto logits = head_scores(p);
    // head_scores_l2h4d128.npy: 128-byte npy header then 8 little-endian doubles
    FILE* f = std::fopen((base + "/head_scores_l2h4d128.npy").c_str(), "rb");
    CHECK(f != nullptr);
    if (f) {
        std::vector<double> want(8);
        std::fseek(f, 128, SEEK_SET);
        CHECK(std::fread(want.data(), 8, 8, f) == 8);
        std::fclose(f);
        for (int i = 0; i < 8; ++i) CHECK(std::fabs(logits[(size_t)i] - want[(size_t)i]) <= 1e-12 * (1.0 + std::fabs(want[(size_t)i])));
    }
    // the checkpoint drives the device path end to end (reference mode, floor budgets)
    BudgetTable t = allocate_budgets(logits, 0.15, 2, 4);
    const int T = 600;
    auto budgets = freeze_budgets(t, T);
    KvTrace tr = make_trace(2, 4, 128, T, 700);
    auto [cache, rep] = prefill_with_eviction(tr, budgets, p.token_scorers, Activation::silu, Precision::bf16);
    for (int h = 0; h < 8; ++h) CHECK(cache.heads[(size_t)h].retained() == budgets[(size_t)h]);
    CHECK_THROWS_AS(load_lkv_params(base + "/does_not_exist.bin"), contract_error);
}

static void test_soft_topk_training() {
    // test_soft_topk.cpp:36-41: four equal scores, k = 1 -> lambda = ln 2
    std::vector<double> z(4, 0.0);
    auto o = soft_topk_forward(z, 1.0, 1.0);
    CHECK(std::fabs(o.threshold_lambda - std::log(2.0)) <= 1e-12);
    for (double v : o.values) CHECK(std::fabs(v - 0.25) <= 1e-12);
    // :43-50: (2, 1, 0) with k = 1.5 -> lambda = 1
    std::vector<double> x{2.0, 1.0, 0.0};
    o = soft_topk_forward(x, 1.5, 1.0);
    CHECK(std::fabs(o.threshold_lambda - 1.0) <= 1e-12);
    double sum = 0.0;
    for (double v : o.values) sum += v;
    CHECK(std::fabs(sum - 1.5) <= 1e-9 * 3);
    // :129-136: unit upstream -> exactly zero score gradient and unit budget gradient
    auto r = uniform(11, -3.0, 3.0, 55);
    o = soft_topk_forward(r, 4.2, 0.7);
    std::vector<double> ones(11, 1.0);
    auto [gx, gk] = soft_topk_vjp(o, ones, 0.7);
    for (double g : gx) CHECK(g == 0.0);
    CHECK(gk == 1.0);
    // :138-170: vjp vs central differences of <u, values>
    auto u = uniform(11, -1.0, 1.0, 72);
    auto [gx2, gk2] = soft_topk_vjp(o, u, 0.7);
    for (int i : {0, 5, 10}) {
        auto xp = r, xm = r;
        xp[(size_t)i] += 1e-5;
        xm[(size_t)i] -= 1e-5;
        auto vp = soft_topk_forward(xp, 4.2, 0.7).values, vm = soft_topk_forward(xm, 4.2, 0.7).values;
        double fd = 0.0;
        for (size_t j = 0; j < 11; ++j) fd += u[j] * (vp[j] - vm[j]) / 2e-5;
        CHECK(std::fabs(fd - gx2[(size_t)i]) <= 1e-6 * (1.0 + std::fabs(fd)));
    }
    // :180-188: n = 1 pins the value to k; vjp (0, 1)
    std::vector<double> one{0.3};
    o = soft_topk_forward(one, 0.4, 1.0);
    CHECK(std::fabs(o.values[0] - 0.4) <= 1e-15);
    std::vector<double> up{2.0};
    auto [g1, k1] = soft_topk_vjp(o, up, 1.0);
    CHECK(g1[0] == 0.0 && k1 == 1.0);
    // clamp_budget: k outside (0, n) -> budget_error; tau <= 0 -> contract_error
    CHECK_THROWS_AS(soft_topk_forward(x, 3.0, 1.0), budget_error);
    CHECK_THROWS_AS(soft_topk_forward(x, 0.0, 1.0), budget_error);
    CHECK_THROWS_AS(soft_topk_forward(x, 1.0, 0.0), contract_error);
    // training_mask: noised scores
    auto g = uniform(11, -1.0, 1.0, 9);
    auto m = training_mask(r, 4.2, 0.7, g, 0.5);
    std::vector<double> rn(11);
    for (size_t i = 0; i < 11; ++i) rn[i] = r[i] + 0.5 * g[i];
    auto ref = soft_topk_forward(rn, 4.2, 0.7);
    for (size_t i = 0; i < 11; ++i) CHECK(std::fabs(m.values[i] - ref.values[i]) <= 1e-12);
}

// fp64 host statement of masked attention + its VJP (attention.cpp:46-201), for the checks below
static void host_attention(const AttentionCall& c, std::vector<double>& out, const std::vector<double>* u,
                           AttentionGrads* g) {
    out.assign((size_t)c.n_q * c.d, 0.0);
    if (g) {
        g->queries.assign((size_t)c.n_q * c.d, 0.0);
        g->keys.assign((size_t)c.t * c.d, 0.0);
        g->values.assign((size_t)c.t * c.d, 0.0);
        g->soft_mask.assign(c.soft_mask.size(), 0.0);
    }
    for (int r = 0; r < c.n_q; ++r) {
        const int pos = c.query_pos_offset + r, end = c.causal ? std::min(c.t, pos + 1) : c.t;
        std::vector<double> s((size_t)end), pr((size_t)end), p((size_t)end);
        double mx = -INFINITY, zr = 0.0, zm = 0.0;
        for (int j = 0; j < end; ++j) {
            double dot = 0.0;
            for (int e = 0; e < c.d; ++e) dot += c.queries[(size_t)r * c.d + e] * c.keys[(size_t)j * c.d + e];
            s[(size_t)j] = c.scale * dot;
            mx = std::max(mx, s[(size_t)j]);
        }
        for (int j = 0; j < end; ++j) zr += (pr[(size_t)j] = std::exp(s[(size_t)j] - mx));
        auto mask_at = [&](int j) {
            return (c.self_always_retained && j == pos) ? 1.0 : (c.soft_mask.empty() ? 1.0 : c.soft_mask[(size_t)j]);
        };
        for (int j = 0; j < end; ++j) {
            pr[(size_t)j] /= zr;
            zm += (p[(size_t)j] = pr[(size_t)j] * mask_at(j));
        }
        for (int j = 0; j < end; ++j) p[(size_t)j] /= zm;
        for (int e = 0; e < c.d; ++e)
            for (int j = 0; j < end; ++j) out[(size_t)r * c.d + e] += p[(size_t)j] * c.values[(size_t)j * c.d + e];
        if (!g) continue;
        const double* ur = u->data() + (size_t)r * c.d;
        std::vector<double> w((size_t)end), ds((size_t)end);
        double wp = 0.0, dpd = 0.0;
        for (int j = 0; j < end; ++j) {
            double acc = 0.0;
            for (int e = 0; e < c.d; ++e) acc += ur[e] * c.values[(size_t)j * c.d + e];
            w[(size_t)j] = acc;
            wp += acc * p[(size_t)j];
        }
        for (int j = 0; j < end; ++j) {
            const double dpt = (w[(size_t)j] - wp) / zm;
            if (!c.soft_mask.empty() && !(c.self_always_retained && j == pos)) g->soft_mask[(size_t)j] += dpt * pr[(size_t)j];
            ds[(size_t)j] = dpt * mask_at(j);
            dpd += ds[(size_t)j] * pr[(size_t)j];
        }
        for (int j = 0; j < end; ++j) {
            const double dsj = pr[(size_t)j] * (ds[(size_t)j] - dpd) * c.scale;
            for (int e = 0; e < c.d; ++e) {
                g->values[(size_t)j * c.d + e] += p[(size_t)j] * ur[e];
                g->queries[(size_t)r * c.d + e] += dsj * c.keys[(size_t)j * c.d + e];
                g->keys[(size_t)j * c.d + e] += dsj * c.queries[(size_t)r * c.d + e];
            }
        }
    }
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 1e-12;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::fabs(a[i] - b[i]));
        den = std::max(den, std::fabs(b[i]));
    }
    return num / den;
}

static void test_masked_attention_training() {
    for (int rep = 0; rep < 6; ++rep) {
        const bool bf = rep >= 3;
        AttentionCall c;
        c.n_q = bf ? 70 : 9;
        c.t = bf ? 150 : 21;
        c.d = bf ? 128 : 16;
        c.queries = uniform((size_t)c.n_q * c.d, -1.0, 1.0, 100 + rep);
        c.keys = uniform((size_t)c.t * c.d, -1.0, 1.0, 200 + rep);
        c.values = uniform((size_t)c.t * c.d, -1.0, 1.0, 300 + rep);
        if (rep % 3 != 2) {
            c.soft_mask = uniform((size_t)c.t, 0.0, 1.0, 400 + rep);
            c.soft_mask[0] = 1.0;
        }
        c.causal = rep % 3 != 1;
        c.query_pos_offset = c.causal ? c.t - c.n_q : 0;
        c.self_always_retained = rep % 2 == 1;
        c.scale = 1.0 / std::sqrt((double)c.d);
        if (bf) {  // the device sees bf16 inputs: compare on the same rounded values
            for (auto* v : {&c.queries, &c.keys, &c.values})
                for (double& e : *v) e = bf16(e);
        }
        auto u = uniform((size_t)c.n_q * c.d, -1.0, 1.0, 500 + rep);
        if (bf)
            for (double& e : u) e = bf16(e);
        AttentionSaved sv;
        auto out = masked_attention_dense(c, &sv, bf ? Precision::bf16 : Precision::fp32);
        auto g = masked_attention_vjp(c, sv, u);
        std::vector<double> ref;
        AttentionGrads rg;
        host_attention(c, ref, &u, &rg);
        const double tol = bf ? 1e-2 : 1e-5;  // north_star: 1e-2 bf16, 1e-5 fp32
        CHECK(max_rel(out, ref) <= tol);
        CHECK(max_rel(g.queries, rg.queries) <= tol);
        CHECK(max_rel(g.keys, rg.keys) <= tol);
        CHECK(max_rel(g.values, rg.values) <= tol);
        if (!c.soft_mask.empty()) CHECK(max_rel(g.soft_mask, rg.soft_mask) <= tol);
    }
    // attention.cpp:82-84: a row without masked mass -> degenerate_mask_error
    AttentionCall c;
    c.n_q = 2;
    c.t = 4;
    c.d = 8;
    c.queries = uniform(16, -1, 1, 1);
    c.keys = uniform(32, -1, 1, 2);
    c.values = uniform(32, -1, 1, 3);
    c.soft_mask.assign(4, 0.0);
    c.scale = 0.3;
    CHECK_THROWS_AS(masked_attention_dense(c), degenerate_mask_error);
    c.soft_mask[1] = -0.5;  // attention.cpp:40-42
    CHECK_THROWS_AS(masked_attention_dense(c), contract_error);
    c.soft_mask.assign(3, 1.0);
    CHECK_THROWS_AS(masked_attention_dense(c), contract_error);
}

int main(int argc, char** argv) {
    try {
        require_b200();
        test_checkpoint(argc > 1 ? argv[1] : nullptr);
        test_budgets();
        test_budget_csv();
        test_hard_topk();
        test_token_scores();
        test_cache_and_prefill();
        test_decode();
        test_memory();
        test_soft_topk_training();
        test_masked_attention_training();
    } catch (const std::exception& e) {
        std::printf("UNCAUGHT %s\n", e.what());
        return 2;
    }
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
