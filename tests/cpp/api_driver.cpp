// api_driver -- runs one scenario through the declaration-compatible API (include/lkv/) on the
// B200 and prints every output as text, for tests/test_reference_api.py to compare with the
// reference's OWN compiled code (oracle/_ref) on identical inputs.
//   api_driver L Hq Hkv d vocab max_len seed | tokens t0 t1 ... | budgets b0 b1 ... |
//              select K | lkv_seed S | sim_seed S | decode k0 k1 ...
// prints: "logits r v0 v1 ..." (forward_full), "head i len p0 p1 ...", "key i v..." (row-major
// retained keys), "val i v...", "report ops peak full compressed", "dlogits s v0 v1 ..." (decode
// steps over the prefill's compacted cache).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lkv/evictsim.hpp"
#include "lkv/model.hpp"
#include "lkv/policy.hpp"

using namespace lkv;

int main(int argc, char** argv) {
    if (argc < 8) return 2;
    ModelConfig c;
    c.n_layers = std::atoi(argv[1]);
    c.n_query_heads = std::atoi(argv[2]);
    c.n_kv_heads = std::atoi(argv[3]);
    c.head_dim = std::atoi(argv[4]);
    c.vocab_size = std::atoi(argv[5]);
    c.max_seq_len = std::atoi(argv[6]);
    c.rng_seed = std::strtoull(argv[7], nullptr, 10);
    std::vector<int> tokens, budgets, decode;
    int select = 0;
    unsigned long long lkv_seed = 1, sim_seed = 1;
    std::vector<int>* cur = nullptr;
    for (int i = 8; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "tokens") cur = &tokens;
        else if (a == "budgets") cur = &budgets;
        else if (a == "decode") cur = &decode;
        else if (a == "select") select = std::atoi(argv[++i]), cur = nullptr;
        else if (a == "lkv_seed") lkv_seed = std::strtoull(argv[++i], nullptr, 10), cur = nullptr;
        else if (a == "sim_seed") sim_seed = std::strtoull(argv[++i], nullptr, 10), cur = nullptr;
        else if (cur) cur->push_back(std::atoi(a.c_str()));
    }
    ModelWeights w = init_model(c);
    ForwardTrace tr = forward_full(w, tokens);
    const int t = (int)tokens.size();
    for (int r = 0; r < t; ++r) {
        std::printf("logits %d", r);
        for (int v = 0; v < c.vocab_size; ++v) std::printf(" %.17g", tr.logits.data()[(size_t)r * c.vocab_size + v]);
        std::printf("\n");
    }
    LkvParams params = init_lkv_params(c, lkv_seed);
    EvictionPolicy pol;
    const SelectKind kinds[] = {SelectKind::learned, SelectKind::random, SelectKind::recency, SelectKind::sink_recent,
                                SelectKind::attn_window};
    pol.select = kinds[select];
    pol.params = &params;
    auto [cache, rep] = prefill_with_eviction(w, tokens, budgets, pol, sim_seed);
    for (size_t i = 0; i < cache.heads.size(); ++i) {
        const HeadCache& h = cache.heads[i];
        std::printf("head %zu %d", i, h.retained());
        for (int p : h.retained_positions) std::printf(" %d", p);
        std::printf("\nkey %zu", i);
        for (double v : h.keys) std::printf(" %.17g", v);
        std::printf("\nval %zu", i);
        for (double v : h.values) std::printf(" %.17g", v);
        std::printf("\n");
    }
    std::printf("report %lld %lld %.17g %.17g\n", (long long)rep.scoring_ops, (long long)rep.peak_kv_values,
                rep.kv_bytes_full, rep.kv_bytes_compressed);
    for (size_t s = 0; s < decode.size(); ++s) {
        std::vector<double> lg = decode_step(w, cache, decode[s]);
        std::printf("dlogits %zu", s);
        for (double v : lg) std::printf(" %.17g", v);
        std::printf("\n");
    }
    return 0;
}
