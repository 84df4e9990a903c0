// subvocab/static_builder.hpp — the static task vocabulary TYPE only.
//
// The offline static builder (Algorithm 1: input-aware / language / tolerance
// filters, /root/reference/proj/src/static_builder.cpp) is outside the
// tailored-head hot path this build replaces. The
// hot path needs only the StaticTaskVocab value it produces, for the
// select(ids, StaticTaskVocab, V) overload (selector.hpp:30-31), so the type
// is declared here with the reference's field layout
// (/root/reference/proj/include/subvocab/static_builder.hpp:33-50).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <optional>
#include <vector>

#include "subvocab/token_set.hpp"

namespace subvocab {

enum class Provenance : std::uint8_t {
    Filtered,    // survived the filter stages
    AlwaysKeep,  // protected token
};

struct StaticTaskVocab {
    TokenSet members;
    std::array<std::size_t, 4> stage_sizes{};  // candidates, input-aware, +language, final
    std::uint64_t pruned_df_sum = 0;
    double tau = 0.0;
    std::optional<std::vector<int>> allowed_blocks;
    std::vector<TokenId> tolerance_pruned;
    std::map<TokenId, Provenance> provenance;
};

}  // namespace subvocab
