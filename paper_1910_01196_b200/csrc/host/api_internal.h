// api_internal.h -- helpers shared by the C++ API translation units
// (locload_api.cpp, pipeline_api.cpp): status -> reference exception, and the
// calling thread's context on the current CUDA device.
#pragma once

#include "locload_b200.h"

namespace locload {
namespace detail {

// LL_ERR_INVALID -> std::invalid_argument, anything else -> std::runtime_error,
// with ll_last_error()'s text
void check(int status);

// this thread's ll_ctx (own stream and scratch) on the current device
ll_ctx* ctx();

} // namespace detail
} // namespace locload
