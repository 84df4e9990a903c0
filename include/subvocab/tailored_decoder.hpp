// subvocab/tailored_decoder.hpp — the device-resident batched API (drop-in
// extension). The reference API in head.hpp/selector.hpp is per plan and by
// value; an inference runtime serving many requests keeps the full head in
// HBM and drives one micro-batch of per-request plans through
//   prepare(): select (a) + plan layout + lane-interleaved gather (b)
//   step():    fused exact-order logits + argmax + remap (c, d)
// without re-uploading weights. Wraps the svt_session_* C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "subvocab/head.hpp"
#include "subvocab/selector.hpp"
#include "subvocab/token_set.hpp"

struct svt_session;

namespace subvocab {

class TailoredDecoder {
public:
    // `head` must outlive the decoder (its device mirror is used in place).
    TailoredDecoder(const HeadMatrix& head, std::size_t max_batch);
    ~TailoredDecoder();
    TailoredDecoder(const TailoredDecoder&) = delete;
    TailoredDecoder& operator=(const TailoredDecoder&) = delete;

    // One plan per prompt: S_b = T ∪ prompt_b. IntegrityError as select().
    void prepare(const TokenSet& static_members, std::span<const std::vector<TokenId>> prompts);

    // One greedy decode step for every prepared request: `hidden` holds
    // batch x dim floats (row b = request b). Returns the global token ids.
    std::vector<TokenId> step(std::span<const float> hidden);

    std::vector<SelectionPlan> plans() const;
    std::size_t batch() const { return batch_; }

private:
    svt_session* session_ = nullptr;
    const HeadMatrix* head_ = nullptr;
    std::size_t batch_ = 0;
};

}  // namespace subvocab
