// subvocab/plan_json.hpp — (f1) the plan wire format of the B200 drop-in.
//
// The reference exposes it through nlohmann::json in
// /root/reference/proj/include/subvocab/artifacts.hpp:24-25
// (to_json(const SelectionPlan&), plan_from_json(const json&, origin)); the
// CLI writes one compact object per line (subvocab.cpp:413) and save_json
// writes dump(2) (artifacts.cpp:249-254). These string-level equivalents
// produce the same bytes without a JSON dependency and throw the same error
// classes (ParseError: malformed / missing field; IntegrityError: ids not
// strictly increasing or out of range), so plans the GPU selects can be
// written for — and read back from — the reference's tools.
#pragma once

#include <string>
#include <string_view>
#include <vector>

#include "subvocab/selector.hpp"

namespace subvocab::artifacts {

// to_json(plan).dump(indent); indent < 0 = compact (the CLI's plans file line)
std::string plan_to_json_text(const SelectionPlan& plan, int indent = -1);

// plan_from_json(json::parse(text), origin)
SelectionPlan plan_from_json_text(std::string_view text, std::string_view origin);

// one compact line per plan (the CLI's `select --plans-out` file)
std::string plans_to_jsonl(const std::vector<SelectionPlan>& plans);

}  // namespace subvocab::artifacts
