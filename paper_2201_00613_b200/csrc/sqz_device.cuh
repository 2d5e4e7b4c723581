// sqz_device.cuh — device helpers shared by the kernel translation units (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_kernels.cuh"

namespace sqz {

// State of a global Ω for a (possibly sharded) buffer: in-shard from `cur`, else from the
// halo receive buffer (binary search over the sorted needs list).
// Byte offset of an in-shard Ω in a tile-padded state buffer.
__device__ __forceinline__ uint64_t pad_offset(const PadLayout& L, uint64_t om) {
  const uint64_t t = fdiv(L.divK, om);
  return (t - L.tile_lo) * L.Kp + (om - t * L.K);
}

__device__ __forceinline__ uint32_t fetch_cell(const uint8_t* __restrict__ cur, uint64_t om, const HaloView& h) {
  if (om >= h.omega_lo && om < h.omega_hi) return __ldg(cur + pad_offset(h.L, om));
  uint64_t lo = 0, hi = h.nneeds;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    uint64_t v = h.needs[mid];
    if (v < om) lo = mid + 1;
    else hi = mid;
  }
  if (lo < h.nneeds && h.needs[lo] == om && h.recv != nullptr) return h.recv[lo];
  if (h.err) atomicExch(h.err, 1);
  return 0;
}

// State of an out-of-shard Ω from the halo receive buffer (binary search over the sorted
// needs list); a miss sets the error flag and reads as dead.
__device__ __forceinline__ uint32_t halo_fetch(const HaloView& h, uint64_t om) {
  uint64_t lo = 0, hi = h.nneeds;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (h.needs[mid] < om) lo = mid + 1;
    else hi = mid;
  }
  if (lo < h.nneeds && h.needs[lo] == om && h.recv != nullptr) return h.recv[lo];
  if (h.err) atomicExch(h.err, 1);
  return 0;
}

}  // namespace sqz
