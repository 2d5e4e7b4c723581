// sqz_heat.cuh — parameters and launchers of the heat-diffusion workload (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_kernels.cuh"

namespace sqz {

struct HeatParams {
  uint32_t K;               // cells per tile = float4 words per 4-tile chunk
  uint32_t P;               // remote (own cell, neighbour) pairs per tile
  uint32_t stages;          // pipeline stages
  float alpha;              // diffusion number α
  const uint16_t* nbr;      // K x 8 word slots in a chunk's [K state | P pairs] float4 slot
  const uint32_t* pairs;    // P: own cell j | link direction << 16
  const uint32_t* pair_j2;  // P: the neighbour's cell in the neighbour tile
};

size_t heat_smem_bytes(const HeatParams& h, const TileParams& p);
cudaError_t heat_prepare(const HeatParams& h, const TileParams& p, int* occupancy);
cudaError_t launch_heat_step(const HeatParams& h, const TileParams& p, const float* cur, float* next, int grid,
                             cudaStream_t st);
cudaError_t launch_heat_seed(const LevelMaps& full, const TileParams& p, float* u, uint64_t seed, cudaStream_t st);
cudaError_t launch_heat_sum(const float* u, uint64_t n, double* out, cudaStream_t st);

}  // namespace sqz
