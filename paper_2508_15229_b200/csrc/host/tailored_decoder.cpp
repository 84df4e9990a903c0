// tailored_decoder.cpp — batched device-resident decoding over svt_session_*.
#include <string>

#include "common.hpp"
#include "subvocab/tailored_decoder.hpp"

namespace subvocab {

using detail::ok;

TailoredDecoder::TailoredDecoder(const HeadMatrix& head, std::size_t max_batch) : head_(&head) {
    ok(svt_session_create(&session_, head.device_data(),
                          static_cast<svt_dtype>(head.device_dtype()), head.rows(), head.dim(),
                          static_cast<std::int32_t>(max_batch), 0, nullptr));
}

TailoredDecoder::~TailoredDecoder() { svt_session_destroy(session_); }

void TailoredDecoder::prepare(const TokenSet& static_members,
                              std::span<const std::vector<TokenId>> prompts) {
    std::vector<TokenId> flat;
    std::vector<std::int64_t> off{0};
    for (const auto& p : prompts) {
        flat.insert(flat.end(), p.begin(), p.end());
        off.push_back(static_cast<std::int64_t>(flat.size()));
    }
    const auto words = static_members.words();
    ok(svt_session_prepare_host(session_, words.data(), static_members.universe_size(),
                                flat.data(), off.data(), static_cast<std::int32_t>(prompts.size())));
    batch_ = prompts.size();
}

std::vector<TokenId> TailoredDecoder::step(std::span<const float> hidden) {
    if (hidden.size() != batch_ * head_->dim())
        throw IntegrityError("hidden state block has " + std::to_string(hidden.size()) +
                             " values but the batch needs " +
                             std::to_string(batch_ * head_->dim()));
    std::vector<TokenId> ids(batch_);
    if (batch_ == 0) return ids;
    ok(svt_session_greedy_host(session_, hidden.data(), head_->dim(), ids.data(), nullptr));
    return ids;
}

std::vector<SelectionPlan> TailoredDecoder::plans() const {
    std::vector<std::int64_t> na(batch_), ns(batch_), nd(batch_), off(batch_ + 1);
    ok(svt_session_plans_host(session_, na.data(), ns.data(), nd.data(), nullptr, nullptr));
    std::size_t total = 0;
    for (const auto n : na) total += static_cast<std::size_t>(n);
    std::vector<std::uint32_t> ids(total);
    ok(svt_session_plans_host(session_, nullptr, nullptr, nullptr, ids.data(), off.data()));
    std::vector<SelectionPlan> out(batch_);
    for (std::size_t b = 0; b < batch_; ++b) {
        out[b].active_ids.assign(ids.begin() + off[b], ids.begin() + off[b + 1]);
        out[b].n_static = static_cast<std::size_t>(ns[b]);
        out[b].n_dynamic = static_cast<std::size_t>(nd[b]);
        out[b].full_vocab_size = head_->rows();
    }
    return out;
}

}  // namespace subvocab
