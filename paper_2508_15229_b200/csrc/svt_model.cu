// svt_model.cu — host-side byte accounting and the offload overlap model that
// accompany the tailored head (no device work).
//
// memory_report follows head.cpp:219-237: the full embedding stays on the
// host (0 bytes on the device) and only the sub-head is device resident;
// saved_fraction compares against keeping both full tables on the device.
// simulate/breakeven_rows follow offload_sim.cpp:44-87: the sub-head transfer
// over the host link overlaps prefill; only max(0, transfer - prefill) is
// exposed. Errors map to ConfigError exactly where the reference throws.
#include <cmath>
#include <cstdint>
#include <limits>

#include "svt_common.cuh"

namespace {

bool bad_width(int b) { return b != 2 && b != 4; }

svt_status hw_check(double link, double flops, double lat) {
    const double v[3] = {link, flops, lat};
    const char* names[3] = {"link_bandwidth", "device_flops", "host_lookup_latency"};
    for (int i = 0; i < 3; ++i)
        if (!(v[i] > 0.0) || !std::isfinite(v[i])) {
            svt::set_error("%s must be strictly positive; got %f", names[i], v[i]);
            return SVT_ERR_CONFIG;
        }
    return SVT_OK;
}

}  // namespace

extern "C" svt_status svt_memory_report(size_t full_size, size_t dim, int dtype_bytes,
                                        size_t plan_size, svt_memory_report_t* out) {
    if (bad_width(dtype_bytes)) {
        svt::set_error("dtype_bytes must be 2 or 4; got %d", dtype_bytes);
        return SVT_ERR_CONFIG;
    }
    const uint64_t row = static_cast<uint64_t>(dim) * static_cast<uint64_t>(dtype_bytes);
    out->full_head_bytes = static_cast<uint64_t>(full_size) * row;
    out->sub_head_bytes = static_cast<uint64_t>(plan_size) * row;
    out->embedding_bytes_gpu = 0;
    out->embedding_bytes_host = out->full_head_bytes;
    const uint64_t base = out->full_head_bytes + out->embedding_bytes_host;
    const uint64_t kept = out->sub_head_bytes + out->embedding_bytes_gpu;
    out->saved_fraction = base == 0      ? 1.0
                          : kept >= base ? 0.0
                                         : static_cast<double>(base - kept) / static_cast<double>(base);
    return SVT_OK;
}

extern "C" svt_status svt_simulate(double link, double flops, double lat, size_t plan_size,
                                   size_t dim, int dtype_bytes, size_t prompt_len, double fpt,
                                   svt_overlap_timeline_t* out) {
    if (svt_status s = hw_check(link, flops, lat)) return s;
    if (fpt < 0.0 || !std::isfinite(fpt)) {
        svt::set_error("model_flops_per_token must be non-negative");
        return SVT_ERR_CONFIG;
    }
    if (dim == 0) {
        svt::set_error("head dimension must be positive");
        return SVT_ERR_CONFIG;
    }
    if (bad_width(dtype_bytes)) {
        svt::set_error("dtype_bytes must be 2 or 4; got %d", dtype_bytes);
        return SVT_ERR_CONFIG;
    }
    const uint64_t row = static_cast<uint64_t>(dim) * static_cast<uint64_t>(dtype_bytes);
    if (plan_size != 0 && row > std::numeric_limits<uint64_t>::max() / plan_size) {
        svt::set_error("plan byte volume overflows");
        return SVT_ERR_CONFIG;
    }
    const double bytes = static_cast<double>(static_cast<uint64_t>(plan_size) * row);
    out->transfer_time = bytes / link;
    out->prefill_time = static_cast<double>(prompt_len) * fpt / flops;
    out->embedding_time = static_cast<double>(prompt_len) * lat;
    out->exposed_latency =
        out->transfer_time > out->prefill_time ? out->transfer_time - out->prefill_time : 0.0;
    out->hidden = out->exposed_latency == 0.0 ? 1 : 0;
    return SVT_OK;
}

extern "C" svt_status svt_breakeven_rows(double link, double flops, double lat, size_t dim,
                                         int dtype_bytes, size_t prompt_len, double fpt,
                                         size_t* out_rows) {
    svt_overlap_timeline_t t;
    if (svt_status s = svt_simulate(link, flops, lat, 0, dim, dtype_bytes, prompt_len, fpt, &t))
        return s;
    const double prefill = t.prefill_time;
    const double row_bytes = static_cast<double>(dim) * static_cast<double>(dtype_bytes);
    const uint64_t max_rows = std::numeric_limits<uint64_t>::max() /
                              (static_cast<uint64_t>(dim) * static_cast<uint64_t>(dtype_bytes));
    auto hidden = [&](uint64_t k, bool* h) -> svt_status {
        svt_overlap_timeline_t x;
        svt_status s = svt_simulate(link, flops, lat, static_cast<size_t>(k), dim, dtype_bytes,
                                    prompt_len, fpt, &x);
        *h = x.hidden != 0;
        return s;
    };
    // closed form, then walk to the exact boundary of simulate()
    const double est = std::floor(prefill * link / row_bytes);
    uint64_t k = 0;
    if (est > 0) k = est >= static_cast<double>(max_rows) ? max_rows : static_cast<uint64_t>(est);
    bool h = false;
    while (k > 0) {
        if (svt_status s = hidden(k, &h)) return s;
        if (h) break;
        --k;
    }
    while (k < max_rows) {
        if (svt_status s = hidden(k + 1, &h)) return s;
        if (!h) break;
        ++k;
    }
    if (k == max_rows) {
        if (svt_status s = hidden(k, &h)) return s;
        if (h) {
            svt::set_error("breakeven exceeds the representable plan size");
            return SVT_ERR_CONFIG;
        }
    }
    *out_rows = static_cast<size_t>(k);
    return SVT_OK;
}
