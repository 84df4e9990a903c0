// bench_dropin_cfg1.cpp — the reference's own call sequence at BASELINE cfg1
// through the C++ drop-in (include/subvocab -> libsubvocab_b200.so):
//   HeadMatrix::random(128256, 2048, 0x5EED)          (SURVEY §8d inputs)
//   select(prompt, T, V)  -> gather(head, plan)        (selector.cpp:16-43, head.cpp:176-187)
//   64 x greedy_step(sub, h_t, plan)                   (head.cpp:203-217)
// with host vectors in and out, exactly as a C++ caller of the reference
// would write it. Prints one JSON line: select / gather / per-token
// greedy_step wall times (steady_clock, medians over runs) and the ids' hash
// (checked against the oracle by tests/test_dropin_cpp.py).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <set>
#include <vector>

#include "subvocab/head.hpp"
#include "subvocab/selector.hpp"
#include "subvocab/token_set.hpp"

using namespace subvocab;
using Clock = std::chrono::steady_clock;

namespace {
std::uint64_t mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
std::uint64_t splitmix(std::uint64_t seed, std::uint64_t k) {  // output k (0-based)
    return mix(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
}
double us_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::micro>(Clock::now() - t0).count();
}
double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}
}  // namespace

int main(int argc, char** argv) {
    const std::size_t V = 128256, d = 2048, L = 512, nT = 2048;
    const int steps = 64, runs = argc > 1 ? std::atoi(argv[1]) : 5;
    const HeadMatrix head = HeadMatrix::random(V, d, 0x5EED);
    TokenSet T(V);
    for (std::uint64_t k = 0; T.size() < nT; ++k) T.insert(static_cast<TokenId>(splitmix(0x57A7, k) % V));
    std::vector<TokenId> prompt(L);
    for (std::size_t i = 0; i < L; ++i) prompt[i] = static_cast<TokenId>(splitmix(0x9A0, i) % V);
    // hidden states: rows of HeadMatrix::random(steps, d, 0x41DD)
    std::vector<std::vector<float>> hid(steps, std::vector<float>(d));
    for (int t = 0; t < steps; ++t)
        for (std::size_t c = 0; c < d; ++c) {
            const std::uint64_t r = splitmix(0x41DD, static_cast<std::uint64_t>(t) * d + c) >> 40;
            hid[t][c] = static_cast<float>(r) * 0x1p-23f - 1.0f;
        }
    std::vector<double> t_sel, t_gat, t_tok;
    std::uint64_t hash = 0;
    std::vector<TokenId> ids(steps);
    for (int run = 0; run < runs + 1; ++run) {  // run 0 = warm-up
        auto t0 = Clock::now();
        const SelectionPlan plan = select(prompt, T, V);
        const double s = us_since(t0);
        t0 = Clock::now();
        const HeadMatrix sub = gather(head, plan);
        const double g = us_since(t0);
        t0 = Clock::now();
        for (int t = 0; t < steps; ++t) ids[t] = greedy_step(sub, hid[t], plan);
        const double k = us_since(t0) / steps;
        if (run == 0) continue;
        t_sel.push_back(s);
        t_gat.push_back(g);
        t_tok.push_back(k);
        hash = 1469598103934665603ull;
        for (TokenId id : ids) hash = (hash ^ id) * 1099511628211ull;
        if (run == 1) {
            std::fprintf(stderr, "plan %zu rows (n_static %zu, n_dynamic %zu); ids", plan.active_ids.size(),
                         plan.n_static, plan.n_dynamic);
            for (int t = 0; t < 8; ++t) std::fprintf(stderr, " %u", ids[t]);
            std::fprintf(stderr, " ...\n");
        }
    }
    const double tok = median(t_tok);
    std::printf("{\"api\": \"C++ drop-in (subvocab::select / gather / greedy_step, host vectors)\", "
                "\"config\": \"cfg1 V=128256 d=2048 f32, 512-token prompt + 2048 static, 64 steps\", "
                "\"runs\": %d, \"select_us\": %.1f, \"gather_us\": %.1f, \"greedy_step_us\": %.2f, "
                "\"tokens_per_s_decode\": %.1f, \"tokens_per_s_job\": %.1f, \"ids\": [",
                runs, median(t_sel), median(t_gat), tok, 1e6 / tok,
                steps * 1e6 / (median(t_sel) + median(t_gat) + steps * tok));
    for (int t = 0; t < steps; ++t) std::printf("%s%u", t ? ", " : "", ids[t]);
    std::printf("], \"ids_fnv1a\": %llu}\n", static_cast<unsigned long long>(hash));
    return 0;
}
