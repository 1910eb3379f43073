// Library baseline for K1 at scale (tools only, never on the product path): CUB's
// DeviceRadixSort::SortPairs (onesweep) on the same (key, admission index) pairs and the
// same bit range that coe_group_sort sorts.  Built by tools/cub_ab/build.sh into
// tools/cub_ab/libcub_sort.so and timed beside K1 by tools/k12_scale.py.
#include <cstdint>
#include <cub/device/device_radix_sort.cuh>

extern "C" {

// Temporary-storage bytes CUB needs for n pairs.
size_t cub_sort_pairs_scratch_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 32);
  return bytes;
}

int cub_sort_pairs(const uint32_t *keys_in, uint32_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                   int64_t n, int end_bit, void *scratch, size_t scratch_bytes, cudaStream_t stream) {
  return (int)cub::DeviceRadixSort::SortPairs(scratch, scratch_bytes, keys_in, keys_out, vals_in, vals_out, (int)n,
                                              0, end_bit, stream);
}
}
