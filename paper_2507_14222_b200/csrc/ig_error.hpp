// ig_error.hpp — internal error type (never crosses the C-ABI; capi.cu maps it
// to an ig_status).
#pragma once

#include <string>
#include <utility>

namespace igb {

struct Error {
    int status;
    std::string msg;
};

[[noreturn]] inline void fail(int status, std::string msg) { throw Error{status, std::move(msg)}; }

}  // namespace igb
