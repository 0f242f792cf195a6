// Trained-policy ingestion through the declaration-compatible API (include/lkv/checkpoint.hpp):
// a checkpoint written by the reference's OWN save path (tests/golden, tests/golden/make_golden.py)
// loads with lkv::load_lkv_params, its LKV-H logits come from lkv::head_scores on the B200 (printed
// for tests/test_reference_api.py to compare with the reference's own head_scores), and
// save -> load round-trips model and policy checkpoints bit for bit.
//   usage: test_checkpoint_api <lkv_params.bin> <scratch dir>
#include <cstdio>
#include <string>

#include "lkv/checkpoint.hpp"
#include "lkv/errors.hpp"
#include "lkv/policy.hpp"

using namespace lkv;

static int fails = 0;
static void expect(bool ok, const char* what) {
    if (!ok) {
        std::printf("FAIL: %s\n", what);
        ++fails;
    }
}

static bool same(const Tensor& a, const Tensor& b) {
    if (a.shape() != b.shape()) return false;
    for (size_t i = 0; i < a.numel(); ++i)
        if (a.data()[i] != b.data()[i]) return false;
    return true;
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string dir = argv[2];
    LkvParams p = load_lkv_params(argv[1]);
    Tensor s = head_scores(p);
    for (size_t i = 0; i < s.numel(); ++i) std::printf("score %zu %.17g\n", i, s.data()[i]);

    save_lkv_params(dir + "/policy_roundtrip.bin", p);
    LkvParams q = load_lkv_params(dir + "/policy_roundtrip.bin");
    expect(q.n_layers == p.n_layers && q.n_kv_heads == p.n_kv_heads && q.d_e == p.d_e && q.d_head == p.d_head,
           "policy geometry round-trips");
    auto pa = p.named_params(), qa = q.named_params();
    expect(pa.size() == qa.size(), "policy tensor count");
    for (size_t i = 0; i < pa.size() && i < qa.size(); ++i) expect(same(*pa[i].second, *qa[i].second), "policy tensor");

    ModelConfig cfg;
    cfg.n_layers = 2;
    cfg.n_query_heads = 4;
    cfg.n_kv_heads = 2;
    cfg.head_dim = 8;
    cfg.vocab_size = 32;
    cfg.rng_seed = 77;
    ModelWeights w = init_model(cfg);
    w.frozen = true;
    save_model(dir + "/model_roundtrip.bin", w);
    ModelWeights back = load_model(dir + "/model_roundtrip.bin");
    expect(back.frozen && back.config.n_layers == 2 && back.config.vocab_size == 32, "model config round-trips");
    auto wa = w.named_params(), wb = back.named_params();
    for (size_t i = 0; i < wa.size(); ++i) expect(same(*wa[i].second, *wb[i].second), "model tensor");

    bool threw = false;
    try {
        load_lkv_params(dir + "/missing.bin");
    } catch (const contract_error&) {
        threw = true;
    }
    expect(threw, "missing file -> contract_error");

    // export-budgets (tools/lkv.cpp:154-177) from the loaded policy, on the device
    BudgetTable table = allocate_budgets(s, 0.15, p.n_layers, p.n_kv_heads);
    std::vector<int> b = freeze_budgets(table, 1000);
    for (size_t i = 0; i < b.size(); ++i) std::printf("budget %zu %d\n", i, b[i]);
    std::printf("%s\n", fails ? "checkpoint api: FAILED" : "checkpoint api: ok");
    return fails ? 1 : 0;
}
