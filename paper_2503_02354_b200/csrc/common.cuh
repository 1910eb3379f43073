// common.cuh -- shared error plumbing for the CUDA C-ABI (coe_cuda.h).
#pragma once
#include <cuda_runtime.h>

#include <string>

void coe_set_error(const std::string &msg);

// Record a CUDA failure; returns true when e == cudaSuccess.
inline bool coe_cuda_ok(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return true;
  coe_set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return false;
}
