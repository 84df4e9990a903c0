// plan_json.cpp — C++ drop-in over the C-ABI plan wire format (svt_plan_*).
#include "subvocab/plan_json.hpp"

#include "common.hpp"

namespace subvocab::artifacts {

std::string plan_to_json_text(const SelectionPlan& plan, int indent) {
    std::size_t need = 0;
    const uint32_t* ids = plan.active_ids.empty() ? nullptr : plan.active_ids.data();
    detail::ok(svt_plan_to_json(ids, plan.active_ids.size(), plan.n_static, plan.n_dynamic,
                                plan.full_vocab_size, indent, nullptr, 0, &need));
    std::string out(need, '\0');
    detail::ok(svt_plan_to_json(ids, plan.active_ids.size(), plan.n_static, plan.n_dynamic,
                                plan.full_vocab_size, indent, out.data(), need, nullptr));
    out.resize(need - 1);
    return out;
}

SelectionPlan plan_from_json_text(std::string_view text, std::string_view origin) {
    const std::string org(origin);
    std::size_t n = 0;
    detail::ok(svt_plan_from_json(text.data(), text.size(), org.c_str(), nullptr, 0, &n, nullptr,
                                  nullptr, nullptr));
    SelectionPlan plan;
    plan.active_ids.resize(n);
    detail::ok(svt_plan_from_json(text.data(), text.size(), org.c_str(),
                                  n ? plan.active_ids.data() : nullptr, n, &n, &plan.n_static,
                                  &plan.n_dynamic, &plan.full_vocab_size));
    return plan;
}

std::string plans_to_jsonl(const std::vector<SelectionPlan>& plans) {
    std::string out;
    for (const SelectionPlan& p : plans) {
        out += plan_to_json_text(p, -1);
        out += '\n';
    }
    return out;
}

}  // namespace subvocab::artifacts
