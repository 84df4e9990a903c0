// offload_sim.cpp — the analytic overlap model (offload_sim.cpp:11-87 of the
// reference) evaluated through svt_simulate / svt_breakeven_rows.
#include <cmath>
#include <string>

#include "common.hpp"
#include "subvocab/offload_sim.hpp"

namespace subvocab {

using detail::ok;

HardwareModel HardwareModel::illustrative_default() {
    HardwareModel hw;
    hw.link_bandwidth = 16.0e9;
    hw.device_flops = 4.0e12;
    hw.host_lookup_latency = 50e-9;
    return hw;
}

void HardwareModel::validate() const {
    const double v[3] = {link_bandwidth, device_flops, host_lookup_latency};
    const char* name[3] = {"link_bandwidth", "device_flops", "host_lookup_latency"};
    for (int i = 0; i < 3; ++i)
        if (!(v[i] > 0.0) || !std::isfinite(v[i]))
            throw ConfigError(std::string(name[i]) + " must be strictly positive; got " +
                              std::to_string(v[i]));
}

OverlapTimeline simulate(const HardwareModel& hw, std::size_t plan_size, std::size_t dim,
                         int dtype_bytes, std::size_t prompt_len,
                         double model_flops_per_token) {
    hw.validate();
    svt_overlap_timeline_t t;
    ok(svt_simulate(hw.link_bandwidth, hw.device_flops, hw.host_lookup_latency, plan_size, dim,
                    dtype_bytes, prompt_len, model_flops_per_token, &t));
    return OverlapTimeline{t.transfer_time, t.prefill_time, t.embedding_time, t.exposed_latency,
                           t.hidden != 0};
}

std::size_t breakeven_rows(const HardwareModel& hw, std::size_t dim, int dtype_bytes,
                           std::size_t prompt_len, double model_flops_per_token) {
    hw.validate();
    std::size_t rows = 0;
    ok(svt_breakeven_rows(hw.link_bandwidth, hw.device_flops, hw.host_lookup_latency, dim,
                          dtype_bytes, prompt_len, model_flops_per_token, &rows));
    return rows;
}

}  // namespace subvocab
