// htrise-b200 drop-in: the process-wide device context of the header API.
//
// Every compute entry point of the reference headers (tensor algebra,
// truncated_svd, bht_l2r, encode, decode, ht_rise_update, ...) runs on the
// device through include/htrise_cuda.h; this header holds the lazily created
// context they share and maps C-ABI status codes back onto the reference's
// exception types. There is no CPU fallback: without a CUDA device every
// compute call throws std::runtime_error.
#pragma once

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "htrise_cuda.h"

namespace htrise {
namespace device {

[[noreturn]] inline void throw_status(htr_status code, const std::string& msg) {
    switch (code) {
        case HTR_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case HTR_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

/// Process-wide default context on device 0 (or $HTRISE_DEVICE).
class Context {
public:
    static Context& instance() {
        static Context c;
        return c;
    }
    htr_context* get() {
        std::call_once(once_, [this] {
            int dev = 0;
            if (const char* e = std::getenv("HTRISE_DEVICE")) dev = std::atoi(e);
            htr_context* c = nullptr;
            const htr_status st = htr_context_create(dev, &c);
            if (st != HTR_OK) {
                const std::string msg = c ? htr_last_error(c) : "htr_context_create failed";
                htr_context_destroy(c);
                error_ = msg;
                code_ = st;
                return;
            }
            ctx_ = c;
        });
        if (!ctx_) throw_status(code_, error_);
        return ctx_;
    }
    void check(htr_status st) {
        if (st != HTR_OK) throw_status(st, htr_last_error(ctx_));
    }
    ~Context() {
        if (ctx_) htr_context_destroy(ctx_);
    }

private:
    Context() = default;
    std::once_flag once_;
    htr_context* ctx_ = nullptr;
    std::string error_;
    htr_status code_ = HTR_OK;
};

inline htr_context* ctx() { return Context::instance().get(); }
inline void check(htr_status st) { Context::instance().check(st); }

}  // namespace device
}  // namespace htrise
