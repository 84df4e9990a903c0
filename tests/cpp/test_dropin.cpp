// test_dropin.cpp — the drop-in C++ API (include/subvocab) on the B200 path,
// exercised with the reference suite's known answers
// (/root/reference/proj/tests/test_token_set.cpp, test_selector.cpp,
// test_head.cpp, acceptance.cpp criteria 4/6/7). Needs a CUDA device.
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>
#include <set>

#include "mini_test.hpp"
#include "subvocab/error.hpp"
#include "subvocab/head.hpp"
#include "subvocab/offload_sim.hpp"
#include "subvocab/plan_json.hpp"
#include "subvocab/selector.hpp"
#include "subvocab/tailored_decoder.hpp"
#include "subvocab/token_set.hpp"

using namespace subvocab;

namespace {
TokenSet make(std::size_t universe, std::initializer_list<TokenId> ids) {
    TokenSet s(universe);
    for (TokenId id : ids) s.insert(id);
    return s;
}
SelectionPlan plan_of(std::vector<TokenId> ids, std::size_t full) {
    SelectionPlan p;
    p.active_ids = std::move(ids);
    p.n_dynamic = p.active_ids.size();
    p.full_vocab_size = full;
    return p;
}
SelectionPlan synthetic_plan(std::size_t n_static, std::size_t n_dynamic, std::size_t full) {
    SelectionPlan p;
    p.n_static = n_static;
    p.n_dynamic = n_dynamic;
    p.full_vocab_size = full;
    for (std::size_t i = 0; i < n_static + n_dynamic; ++i)
        p.active_ids.push_back(static_cast<TokenId>(i));
    return p;
}
bool same_bits(float a, float b) {
    std::uint32_t x, y;
    std::memcpy(&x, &a, 4);
    std::memcpy(&y, &b, 4);
    return x == y;
}
std::vector<float> rand_hidden(std::mt19937_64& rng, std::size_t d) {
    std::uniform_real_distribution<float> u(-1.0f, 1.0f);
    std::vector<float> h(d);
    for (float& v : h) v = u(rng);
    return h;
}
}  // namespace

// ---- token_set -----------------------------------------------------------------
TEST_CASE("token_set: from_ids deduplicates and algebra holds") {
    CHECK(TokenSet::from_ids(8, std::vector<TokenId>{3, 3, 1}).to_ids() ==
          std::vector<TokenId>({1, 3}));
    CHECK(set_union(make(8, {1, 2}), make(8, {2, 3})).to_ids() == std::vector<TokenId>({1, 2, 3}));
    CHECK(set_intersection(make(8, {1, 2}), make(8, {2, 3})).to_ids() == std::vector<TokenId>({2}));
    CHECK(set_difference(make(8, {1, 2}), make(8, {})).to_ids() == std::vector<TokenId>({1, 2}));
    CHECK_THROWS_AS(set_union(make(8, {1}), make(9, {1})), IntegrityError);
    TokenSet s = make(100, {5, 50, 99});
    s.erase(50);
    s.erase(50);
    CHECK(s.size() == 2);
    std::mt19937_64 rng(0xA11CE);
    for (int it = 0; it < 100; ++it) {
        TokenSet a(64), b(64);
        for (int k = 0; k < 30; ++k) {
            a.insert(static_cast<TokenId>(rng() % 64));
            b.insert(static_cast<TokenId>(rng() % 64));
        }
        CHECK(set_union(a, b) == set_union(b, a));
        CHECK(set_union(set_difference(a, b), set_intersection(a, b)) == a);
        CHECK(a.is_subset_of(set_union(a, b)));
    }
}

// ---- selector --------------------------------------------------------------------
TEST_CASE("selector: fixture plan aca -> [0,2,3,4]") {
    const SelectionPlan plan = select(std::vector<TokenId>{0, 2, 0}, make(8, {3, 4}), 8);
    CHECK(plan.active_ids == std::vector<TokenId>({0, 2, 3, 4}));
    CHECK(plan.n_dynamic == 2);
    CHECK(plan.n_static == 2);
    CHECK(plan.full_vocab_size == 8);
}

TEST_CASE("selector: empty static, input inside static, errors") {
    const SelectionPlan a = select(std::vector<TokenId>{7, 3, 3}, TokenSet(16), 16);
    CHECK(a.active_ids == std::vector<TokenId>({3, 7}));
    CHECK(a.n_dynamic == 2 && a.n_static == 0);
    const SelectionPlan b = select(std::vector<TokenId>{2, 1, 2}, make(8, {1, 2, 5}), 8);
    CHECK(b.n_dynamic == 0);
    CHECK(b.active_ids == std::vector<TokenId>({1, 2, 5}));
    CHECK_THROWS_AS(select(std::vector<TokenId>{8}, TokenSet(8), 8), IntegrityError);
    CHECK_THROWS_AS(select(std::vector<TokenId>{0}, TokenSet(4), 8), IntegrityError);
    try {
        select(std::vector<TokenId>{1, 12, 30}, TokenSet(9), 9);
        CHECK(false);
    } catch (const IntegrityError& e) {
        CHECK(std::string(e.what()).find("input token id 12 ") != std::string::npos);
        CHECK(e.exit_code() == 4);
    }
    StaticTaskVocab v;
    v.members = make(8, {3, 4});
    CHECK(select(std::vector<TokenId>{0, 2}, v, 8).active_ids == std::vector<TokenId>({0, 2, 3, 4}));
}

TEST_CASE("selector: remap_out / global_to_local invert the gather") {
    const SelectionPlan plan = select(std::vector<TokenId>{0, 2}, make(8, {3, 4}), 8);
    CHECK(remap_out(plan, 0) == 0);
    CHECK(remap_out(plan, 3) == 4);
    CHECK_THROWS_AS(remap_out(plan, 4), IntegrityError);
    for (std::size_t k = 0; k < plan.size(); ++k) CHECK(plan.global_to_local(plan.active_ids[k]) == k);
    CHECK(!plan.global_to_local(1).has_value());
}

TEST_CASE("artifacts: plan JSON round-trips and validates (test_artifacts.cpp:44-62)") {
    SelectionPlan plan = plan_of({0, 2, 3, 4}, 8);
    plan.n_static = 2;
    plan.n_dynamic = 2;
    const std::string compact = artifacts::plan_to_json_text(plan);
    CHECK(compact == "{\"active_ids\":[0,2,3,4],\"full_vocab_size\":8,\"n_dynamic\":2,\"n_static\":2}");
    const SelectionPlan back = artifacts::plan_from_json_text(artifacts::plan_to_json_text(plan, 2), "<mem>");
    CHECK(back.active_ids == plan.active_ids);
    CHECK(back.n_static == 2 && back.n_dynamic == 2 && back.full_vocab_size == 8);
    CHECK_THROWS_AS(artifacts::plan_from_json_text(
                        "{\"active_ids\":[2,2],\"full_vocab_size\":8,\"n_dynamic\":2,\"n_static\":2}", "<mem>"),
                    IntegrityError);
    CHECK_THROWS_AS(artifacts::plan_from_json_text(
                        "{\"active_ids\":[2,9],\"full_vocab_size\":8,\"n_dynamic\":2,\"n_static\":2}", "<mem>"),
                    IntegrityError);
    bool named = false;
    try {
        artifacts::plan_from_json_text("{\"active_ids\":[0],\"full_vocab_size\":8,\"n_dynamic\":2}",
                                       "plan.json");
    } catch (const ParseError& e) {
        named = std::string(e.what()).find("plan.json") != std::string::npos;
    }
    CHECK(named);
    CHECK(artifacts::plans_to_jsonl({plan, plan}) == compact + "\n" + compact + "\n");
}

TEST_CASE("selector: reporting convention strings") {
    CHECK(format_vocab_line(18874, 40.0, 151643) == "18,874 + [40] (12.47%)");
    CHECK(format_vocab_line(0, 105.0, 128000) == "[105] (0.08%)");
    CHECK(format_vocab_line(2, 2.0, 8) == "2 + [2] (50.00%)");
    CHECK(format_vocab_line(1234567, 0.4, 2000000) == "1,234,567 + [0] (61.73%)");
    CHECK(format_thousands(0) == "0");
    CHECK(format_thousands(1234567890) == "1,234,567,890");
    std::vector<SelectionPlan> zh{synthetic_plan(18874, 38, 151643), synthetic_plan(18874, 42, 151643)};
    CHECK(batch_stats(zh).line == "18,874 + [40] (12.47%)");
    PlanStats st;
    for (std::size_t d = 1; d <= 100; ++d) st.add(synthetic_plan(0, d, 1000));
    const BatchReport r = st.finalize();
    CHECK(r.p50_active == 50 && r.p90_active == 90 && r.p99_active == 99 && r.max_active == 100);
    CHECK_THROWS_AS(batch_stats({}), ConfigError);
}

TEST_CASE("selector: union_plans on the device") {
    const TokenSet statics = make(8, {5});
    std::vector<SelectionPlan> plans{select(std::vector<TokenId>{0}, statics, 8),
                                     select(std::vector<TokenId>{2, 3}, statics, 8)};
    const SelectionPlan u = union_plans(plans);
    CHECK(u.active_ids == std::vector<TokenId>({0, 2, 3, 5}));
    CHECK(u.n_static == 1 && u.n_dynamic == 3);
    CHECK_THROWS_AS(union_plans({}), ConfigError);
}

// ---- head ------------------------------------------------------------------------
TEST_CASE("head: gather copies the named rows exactly") {
    const HeadMatrix head = HeadMatrix::random(8, 4, 1234);
    const HeadMatrix sub = gather(head, plan_of({0, 2, 3, 4}, 8));
    REQUIRE(sub.rows() == 4 && sub.dim() == 4);
    const std::vector<TokenId> ids{0, 2, 3, 4};
    for (std::size_t k = 0; k < 4; ++k)
        for (std::size_t c = 0; c < 4; ++c) CHECK(same_bits(sub.at(k, c), head.at(ids[k], c)));
    const HeadMatrix h6 = HeadMatrix::random(6, 3, 9);
    CHECK(gather(h6, plan_of({0, 1, 2, 3, 4, 5}, 6)) == h6);
    CHECK(gather(h6, plan_of({}, 6)).rows() == 0);
    CHECK_THROWS_AS(gather(h6, plan_of({6}, 8)), IntegrityError);
}

TEST_CASE("head: logits basics") {
    HeadMatrix head(2, 1, 4);
    head.at(0, 0) = 2.0f;
    head.at(1, 0) = 3.0f;
    CHECK(logits(head, std::vector<float>{5.0f}) == std::vector<float>({10.0f, 15.0f}));
    const HeadMatrix r = HeadMatrix::random(4, 8, 7);
    for (float v : logits(r, std::vector<float>(8, 0.0f))) CHECK(v == 0.0f);
    CHECK_THROWS_AS(logits(r, std::vector<float>{1.0f}), IntegrityError);
}

TEST_CASE("head: sub-head logits equal full-head logits bitwise (acceptance 4)") {
    std::mt19937_64 rng(0x10617);
    for (int it = 0; it < 200; ++it) {
        const std::size_t rows = 1 + rng() % 32, dim = 1 + rng() % 16;
        const HeadMatrix head = HeadMatrix::random(rows, dim, rng());
        std::vector<TokenId> picked;
        for (TokenId r = 0; r < rows; ++r)
            if (rng() & 1) picked.push_back(r);
        const SelectionPlan plan = plan_of(picked, rows);
        const auto h = rand_hidden(rng, dim);
        const auto full = logits(head, h);
        const auto sub = logits(gather(head, plan), h);
        REQUIRE(sub.size() == picked.size());
        for (std::size_t k = 0; k < sub.size(); ++k) CHECK(same_bits(sub[k], full[picked[k]]));
        // and against a host evaluation in the reference order
        for (std::size_t r = 0; r < rows; ++r) {
            float acc = 0.0f;
            for (std::size_t c = 0; c < dim; ++c) {
                volatile float p = head.at(r, c) * h[c];
                acc = acc + p;
            }
            CHECK(same_bits(acc, full[r]));
        }
    }
}

TEST_CASE("head: greedy step decodes through the plan") {
    HeadMatrix sub(3, 1, 4);
    sub.at(0, 0) = 1.0f;
    sub.at(1, 0) = 3.0f;
    sub.at(2, 0) = 2.0f;
    const SelectionPlan plan = plan_of({0, 2, 4}, 8);
    CHECK(greedy_step(sub, std::vector<float>{1.0f}, plan) == 2);
    HeadMatrix flat(3, 1, 4);
    flat.at(0, 0) = flat.at(1, 0) = flat.at(2, 0) = 1.0f;
    CHECK(greedy_step(flat, std::vector<float>{1.0f}, plan) == 0);
    CHECK_THROWS_AS(greedy_step(HeadMatrix(0, 1, 4), std::vector<float>{1.0f}, plan_of({}, 8)),
                    IntegrityError);
    std::mt19937_64 rng(0xA26A);
    for (int it = 0; it < 100; ++it) {
        const HeadMatrix head = HeadMatrix::random(16, 8, rng());
        std::vector<TokenId> picked;
        for (TokenId r = 0; r < 16; ++r)
            if (rng() & 1) picked.push_back(r);
        if (picked.empty()) continue;
        const SelectionPlan p = plan_of(picked, 16);
        const auto h = rand_hidden(rng, 8);
        const auto full = logits(head, h);
        std::size_t arg = 0;
        for (std::size_t r = 1; r < 16; ++r)
            if (full[r] > full[arg]) arg = r;
        const TokenId got = greedy_step(gather(head, p), h, p);
        if (p.global_to_local(static_cast<TokenId>(arg))) CHECK(got == arg);
    }
}

TEST_CASE("head: top-k extension (value desc, id asc; element 0 == greedy_step)") {
    HeadMatrix sub(5, 1, 4);
    sub.at(0, 0) = 1.0f;
    sub.at(1, 0) = 3.0f;
    sub.at(2, 0) = 2.0f;
    sub.at(3, 0) = 3.0f;  // ties row 1: the lower id first
    sub.at(4, 0) = -1.0f;
    const SelectionPlan plan = plan_of({0, 2, 4, 6, 9}, 16);
    const auto top = topk_step(sub, std::vector<float>{1.0f}, plan, 4);
    CHECK((top == std::vector<TokenId>{2, 6, 4, 0}));
    CHECK(topk_step(sub, std::vector<float>{1.0f}, plan, 9).size() == 5);
    CHECK_THROWS_AS(topk_step(sub, std::vector<float>{1.0f}, plan, 0), ConfigError);
    std::mt19937_64 rng(0x70CC);
    for (int it = 0; it < 50; ++it) {
        const HeadMatrix head = HeadMatrix::random(300, 16, rng());
        std::vector<TokenId> picked;
        for (TokenId r = 0; r < 300; ++r)
            if (rng() & 1) picked.push_back(r);
        if (picked.empty()) continue;
        const SelectionPlan p = plan_of(picked, 300);
        const auto h = rand_hidden(rng, 16);
        const HeadMatrix g = gather(head, p);
        const auto k = topk_step(g, h, p, 8);
        CHECK(k.front() == greedy_step(g, h, p));
        const auto lg = logits(g, h);
        for (std::size_t j = 1; j < k.size(); ++j) {
            const float a = lg[*p.global_to_local(k[j - 1])], b = lg[*p.global_to_local(k[j])];
            CHECK((a > b || (a == b && k[j - 1] < k[j])));
        }
    }
}

TEST_CASE("head: memory report arithmetic") {
    const MemoryReport r = memory_report(128000, 2048, 2, 105);
    CHECK(r.sub_head_bytes == 430080);
    CHECK(r.full_head_bytes == 524288000ULL);
    CHECK(r.embedding_bytes_gpu == 0);
    CHECK(r.saved_fraction > 0.99);
    CHECK(memory_report(1000, 64, 4, 1000).saved_fraction == 0.5);
    CHECK(memory_report(1000, 64, 4, 0).saved_fraction == 1.0);
    CHECK_THROWS_AS(memory_report(10, 10, 3, 1), ConfigError);
}

TEST_CASE("head: weight files round-trip bit-exactly (device loader)") {
    const auto dir = std::filesystem::temp_directory_path() / "svt_dropin_test";
    std::filesystem::create_directories(dir);
    const HeadMatrix m32 = HeadMatrix::random(16, 8, 42, 4);
    m32.save(dir / "w.bin");
    CHECK(HeadMatrix::load(dir / "w.bin") == m32);
    const HeadMatrix m16 = HeadMatrix::random(16, 8, 42, 2);
    m16.save(dir / "w16.bin");
    const HeadMatrix back = HeadMatrix::load(dir / "w16.bin");
    CHECK(back == m16);
    CHECK(back.dtype_bytes() == 2);
    // the loaded f16 head decodes like the host-built one
    std::mt19937_64 rng(7);
    const auto h = rand_hidden(rng, 8);
    const auto a = logits(back, h), b = logits(m16, h);
    for (std::size_t i = 0; i < a.size(); ++i) CHECK(same_bits(a[i], b[i]));
    {
        std::ofstream f(dir / "junk.bin");
        f << "definitely not a weight file";
    }
    CHECK_THROWS_AS(HeadMatrix::load(dir / "junk.bin"), ParseError);
    std::filesystem::remove_all(dir);
}

TEST_CASE("head: half conversion round-trips every non-NaN pattern") {
    for (std::uint32_t h = 0; h <= 0xFFFF; ++h) {
        const auto half = static_cast<std::uint16_t>(h);
        if (((half >> 10) & 0x1F) == 0x1F && (half & 0x3FF)) continue;
        CHECK(float_to_half(half_to_float(half)) == half);
    }
    CHECK(half_to_float(0x3C00) == 1.0f);
    CHECK(float_to_half(0.5f) == 0x3800);
}

// ---- offload model ---------------------------------------------------------------
TEST_CASE("offload: simulate and breakeven agree") {
    const HardwareModel hw = HardwareModel::illustrative_default();
    const std::size_t k = breakeven_rows(hw, 2048, 2, 512, 2e9);
    CHECK(simulate(hw, k, 2048, 2, 512, 2e9).hidden);
    CHECK(!simulate(hw, k + 1, 2048, 2, 512, 2e9).hidden);
    HardwareModel bad = hw;
    bad.device_flops = 0.0;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
}

// ---- batched device decoder ---------------------------------------------------------
TEST_CASE("tailored decoder: batched step == per-plan greedy_step") {
    const std::size_t V = 5000, d = 256, B = 6;
    const HeadMatrix head = HeadMatrix::random(V, d, 0x5EED);
    std::mt19937_64 rng(99);
    TokenSet T(V);
    for (int i = 0; i < 300; ++i) T.insert(static_cast<TokenId>(rng() % V));
    std::vector<std::vector<TokenId>> prompts(B);
    for (auto& p : prompts)
        for (int i = 0; i < 80; ++i) p.push_back(static_cast<TokenId>(rng() % V));
    TailoredDecoder dec(head, B);
    dec.prepare(T, prompts);
    const auto plans = dec.plans();
    REQUIRE(plans.size() == B);
    std::vector<float> hidden;
    for (std::size_t b = 0; b < B; ++b) {
        const auto h = rand_hidden(rng, d);
        hidden.insert(hidden.end(), h.begin(), h.end());
    }
    const auto ids = dec.step(hidden);
    for (std::size_t b = 0; b < B; ++b) {
        const SelectionPlan want = select(prompts[b], T, V);
        CHECK(plans[b].active_ids == want.active_ids);
        CHECK(plans[b].n_dynamic == want.n_dynamic);
        const std::span<const float> hb(hidden.data() + b * d, d);
        CHECK(ids[b] == greedy_step(gather(head, want), hb, want));
    }
    std::vector<std::vector<TokenId>> bad{{static_cast<TokenId>(V)}};
    CHECK_THROWS_AS(dec.prepare(T, bad), IntegrityError);
}

int main() { return mini::run_all(); }
