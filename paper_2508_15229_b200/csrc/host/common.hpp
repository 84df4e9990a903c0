// common.hpp — shared plumbing of the C++ drop-in (not installed).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>

#include "subvocab/error.hpp"
#include "svt.h"

namespace subvocab::detail {

inline std::string last_error() {
    const char* m = svt_last_error();
    return m ? std::string(m) : std::string();
}

// Raise the exception matching an svt_status, with the library's message.
inline void ok(svt_status s) {
    if (s != SVT_OK) raise_status(s, last_error());
}

// Owning device allocation (long-lived objects: head mirrors, sub-heads).
struct DeviceBuffer {
    void* ptr = nullptr;
    std::size_t bytes = 0;

    explicit DeviceBuffer(std::size_t n) : bytes(n) { ok(svt_device_alloc(&ptr, n ? n : 16)); }
    ~DeviceBuffer() { svt_device_free(ptr); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;

    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
    void upload(const void* host, std::size_t n) { ok(svt_memcpy_h2d(ptr, host, n, nullptr)); }
    void download(void* host, std::size_t n) const {
        ok(svt_memcpy_d2h(host, ptr, n, nullptr));
        ok(svt_stream_synchronize(nullptr));
    }
};

// Per-thread, per-device scratch for the by-value API calls (select, gather,
// logits, greedy_step, union_plans): device buffers that only grow, a pinned
// host staging area and the thread's own non-blocking stream. A call stages
// its inputs through pinned memory, runs its kernels on the thread's stream
// and synchronises that stream once — no cudaMalloc/cudaFree per call, no
// device-wide synchronisation, and concurrent callers on different threads
// never share buffers (the reference API is reentrant).
class Scratch {
public:
    enum Slot { kIn0, kIn1, kIn2, kOut0, kOut1, kMeta, kWork, kRowsWs, kSlots };

    static Scratch& get();  // this thread's scratch on the current device
    ~Scratch();
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;

    // device buffer of slot s with at least `bytes` (contents undefined, except
    // kRowsWs, which is zeroed whenever it is (re)allocated: the certified
    // rows kernel keeps its control words consistent from then on)
    void* dev(Slot s, std::size_t bytes);
    // pinned host staging of at least `bytes` (one area, reused per call)
    void* host(std::size_t bytes);
    svt_stream stream();

    // host -> device through the pinned area (async on the thread's stream;
    // the staging copy is complete when this returns, so `src` may change)
    void* upload(Slot s, const void* src, std::size_t bytes);
    // device -> host: async copies into pinned staging, one stream sync, then
    // memcpy out. dsts/srcs/bytes are parallel arrays of n entries.
    void download(std::size_t n, void* const* dsts, const void* const* srcs,
                  const std::size_t* bytes);
    void sync() { ok(svt_stream_synchronize(stream())); }

private:
    void* dev_[kSlots] = {};
    std::size_t cap_[kSlots] = {};
    void* pinned_ = nullptr;
    std::size_t pinned_cap_ = 0;
    std::size_t pinned_used_ = 0;  // uploads since the last sync share the area
    svt_stream stream_ = nullptr;
    int device_ = -1;
};

}  // namespace subvocab::detail
