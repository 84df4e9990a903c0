// scratch.cpp — per-thread reusable device / pinned buffers and stream of the
// C++ drop-in (common.hpp: Scratch).
#include <algorithm>
#include <map>
#include <memory>

#include "common.hpp"

namespace subvocab::detail {

namespace {
constexpr std::size_t align_up(std::size_t n) { return (n + 255) & ~std::size_t(255); }
}  // namespace

Scratch& Scratch::get() {
    thread_local std::map<int, std::unique_ptr<Scratch>> per_device;
    int dev = 0;
    ok(svt_get_device(&dev));
    auto& s = per_device[dev];
    if (!s) {
        s = std::make_unique<Scratch>();
        s->device_ = dev;
    }
    return *s;
}

Scratch::~Scratch() {
    // (at process exit the runtime may be gone already: errors are ignored)
    if (stream_) svt_stream_synchronize(stream_);
    for (void*& p : dev_)
        if (p) svt_device_free(p);
    if (pinned_) svt_host_free_pinned(pinned_);
    if (stream_) svt_stream_destroy(stream_);
}

svt_stream Scratch::stream() {
    if (!stream_) ok(svt_stream_create(&stream_));
    return stream_;
}

void* Scratch::dev(Slot s, std::size_t bytes) {
    bytes = std::max<std::size_t>(bytes, 16);
    if (cap_[s] < bytes) {
        // the buffer may still be read by queued work of an earlier call
        if (dev_[s]) {
            sync();
            ok(svt_device_free(dev_[s]));
            dev_[s] = nullptr;
            cap_[s] = 0;
        }
        const std::size_t want = std::max(align_up(bytes), 2 * cap_[s]);
        ok(svt_device_alloc(&dev_[s], want));
        cap_[s] = want;
        if (s == kRowsWs) ok(svt_memset(dev_[s], 0, want, stream()));
    }
    return dev_[s];
}

void* Scratch::host(std::size_t bytes) {
    if (pinned_cap_ < bytes) {
        if (pinned_) {
            sync();  // queued copies may still read the old area
            ok(svt_host_free_pinned(pinned_));
            pinned_ = nullptr;
        }
        const std::size_t want = std::max(align_up(bytes), 2 * pinned_cap_);
        ok(svt_host_alloc_pinned(&pinned_, want));
        pinned_cap_ = want;
        pinned_used_ = 0;
    }
    return pinned_;
}

void* Scratch::upload(Slot s, const void* src, std::size_t bytes) {
    void* d = dev(s, bytes);
    if (bytes == 0) return d;
    if (pinned_used_ + align_up(bytes) > pinned_cap_) {
        sync();  // earlier staged uploads have landed
        pinned_used_ = 0;
        host(align_up(bytes));
    }
    char* stage = static_cast<char*>(pinned_) + pinned_used_;
    std::memcpy(stage, src, bytes);
    ok(svt_memcpy_h2d(d, stage, bytes, stream()));
    pinned_used_ += align_up(bytes);
    return d;
}

void Scratch::download(std::size_t n, void* const* dsts, const void* const* srcs,
                       const std::size_t* bytes) {
    std::size_t total = 0;
    for (std::size_t i = 0; i < n; ++i) total += align_up(bytes[i]);
    if (pinned_used_ + total > pinned_cap_) {
        sync();
        pinned_used_ = 0;
        host(total);
    }
    char* base = static_cast<char*>(pinned_) + pinned_used_;
    std::size_t at = 0;
    for (std::size_t i = 0; i < n; ++i) {
        if (bytes[i]) ok(svt_memcpy_d2h(base + at, srcs[i], bytes[i], stream()));
        at += align_up(bytes[i]);
    }
    sync();
    at = 0;
    for (std::size_t i = 0; i < n; ++i) {
        if (bytes[i]) std::memcpy(dsts[i], base + at, bytes[i]);
        at += align_up(bytes[i]);
    }
    pinned_used_ = 0;
}

}  // namespace subvocab::detail
