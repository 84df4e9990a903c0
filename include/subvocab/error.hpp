// subvocab/error.hpp — exception taxonomy of the drop-in (B200 build).
//
// Same classes and process exit codes as the reference
// (/root/reference/proj/include/subvocab/error.hpp:10-38), so callers that
// catch subvocab::IntegrityError etc. keep working. The C-ABI status codes of
// include/svt.h are these exit codes; detail::raise() turns one into the
// matching exception.
#pragma once

#include <stdexcept>
#include <string>

namespace subvocab {

// Base class; exit code 1 (also used for CUDA / runtime failures).
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
    virtual int exit_code() const { return 1; }
};

// Invalid configuration (bad dtype width, non-positive hardware figure, empty
// union batch ...): exit code 2.
class ConfigError : public Error {
public:
    using Error::Error;
    int exit_code() const override { return 2; }
};

// Malformed input data (weight files): exit code 3.
class ParseError : public Error {
public:
    using Error::Error;
    int exit_code() const override { return 3; }
};

// Inconsistent artifacts (ids out of range, mismatched vocabularies or plan
// sizes): exit code 4.
class IntegrityError : public Error {
public:
    using Error::Error;
    int exit_code() const override { return 4; }
};

namespace detail {
// Throw the exception class matching a C-ABI status (no-op for 0).
[[noreturn]] void raise_status(int status, const std::string& message);
inline void check_status(int status, const std::string& message) {
    if (status != 0) raise_status(status, message);
}
}  // namespace detail

}  // namespace subvocab
