// common.hpp — shared plumbing of the C++ drop-in (not installed).
#pragma once

#include <cstddef>
#include <cstdint>
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

// Owning device allocation.
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

}  // namespace subvocab::detail
