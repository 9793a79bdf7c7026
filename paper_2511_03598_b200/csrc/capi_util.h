// capi_util.h — shared pieces of the extern "C" boundary (capi.cu,
// sketch_api.cu): exception -> ttr_status mapping, per-thread last error,
// device selection per context, handle helpers.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "tt_round.h"

extern thread_local std::string g_last_error;

namespace ttr {
namespace capi {

template <typename F>
inline ttr_status guard(F&& f) {
    try {
        f();
        return TTR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return TTR_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_last_error = std::string("internal: ") + e.what();
        return TTR_ERR_INTERNAL;
    }
}

inline void need(bool ok, const char* what) {
    if (!ok) throw Error(TTR_ERR_INVALID_ARGUMENT, std::string("InvalidArgument: ") + what);
}

// Entry points bound to a context run on its device (the caller's current
// device may be another one, e.g. a second context in the same process).
template <typename F>
inline ttr_status guard_ctx(ttr_ctx* ctx, F&& f) {
    return guard([&] {
        if (ctx) {
            int cur = -1;
            TTR_CUDA(cudaGetDevice(&cur));
            if (cur != ctx->c.device) TTR_CUDA(cudaSetDevice(ctx->c.device));
        }
        f();
    });
}

inline std::vector<i64> vec(const int64_t* p, int64_t n) { return std::vector<i64>(p, p + n); }

inline ttr_tt* wrap(std::unique_ptr<TTDev> t) {
    auto* o = new ttr_tt;
    o->t = std::move(t);
    return o;
}

inline void check_same_ctx(ttr_ctx* ctx, const ttr_tt* t) {
    need(ctx && t && t->t, "null handle");
    need(t->t->ctx == &ctx->c, "tensor belongs to another context");
}
}  // namespace capi
}  // namespace ttr
