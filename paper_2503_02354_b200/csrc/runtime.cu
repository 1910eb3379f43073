// runtime.cu -- GPU serving runtime (placeholder: error plumbing only).
#include <string>

#include "coe_cuda.h"
#include "common.cuh"

namespace {
thread_local std::string g_last_error;
}

void coe_set_error(const std::string &msg) { g_last_error = msg; }

extern "C" const char *coe_cuda_last_error(void) { return g_last_error.c_str(); }
