// sqz_mma.cu — tensor-core ablation of the ν map.
//
// The paper evaluates ν as a matrix product: per coordinate, the replica ids H_ν[θ_μ] of its
// levels form a row of A, the per-level weights form B, and D = A·B is the compact index
// (its FP16 form is exact only while the weights stay <= 2048, reading D14).  This
// build keeps the map exact with an INTEGER product: Ω = Σ_μ H_ν[θ_μ] k^{μ−1} (D2) is
//
//     D[c][b] = Σ_μ A[c][μ] · B[μ][b],   A[c][μ] = H_ν[θ_μ(c)] (u8),  B[μ][b] = byte b of k^{μ−1},
//     Ω(c)    = Σ_b D[c][b] · 256^b,
//
// one mma.sync.m16n8k32 u8 x u8 -> s32 per 16 coordinates (M = 16 coordinates, K = 32 levels,
// N = 8 weight bytes).  A hole at any level (H = HOLE) or a coordinate outside [0, s^r)² gives
// UINT64_MAX, as squeeze_map_nu does.  It is an ablation: bench.py times it beside the LUT map
// (k_map_nu), and the hot path keeps the LUT.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_kernels.cuh"

namespace sqz {

__global__ void __launch_bounds__(256) k_map_nu_mma(MmaNuParams q, const uint32_t* __restrict__ xi,
                                                    const uint32_t* __restrict__ yi, uint64_t* __restrict__ om,
                                                    uint64_t count) {
  __shared__ int16_t s_h[kMmaMaxS2];  // H_ν[θy * s + θx], -1 = hole
  __shared__ uint32_t s_pw[32];       // s^(μ-1)
  for (uint32_t i = threadIdx.x; i < q.s * q.s; i += blockDim.x) s_h[i] = q.hnu[i];
  if (threadIdx.x < 32) {
    uint32_t v = 1;
    for (uint32_t m = 0; m < threadIdx.x && m < q.r; ++m) v *= q.s;
    s_pw[threadIdx.x] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t g = (uint32_t)lane >> 2, t = (uint32_t)lane & 3u;
  // B fragment (K x N = 32 levels x 8 bytes, column-major): b0 rows 4t..4t+3, b1 rows 16+4t.., col g
  uint32_t b0 = 0, b1 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    b0 |= (uint32_t)q.B[(4 * t + i) * 8 + g] << (8 * i);
    b1 |= (uint32_t)q.B[(16 + 4 * t + i) * 8 + g] << (8 * i);
  }
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t s = q.s;

  // A entries of one coordinate at levels l0..l0+3 (packed u8) and the hole flag
  auto levels = [&](uint32_t x, uint32_t y, uint32_t l0, bool& hole) -> uint32_t {
    uint32_t a = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t l = l0 + i;
      if (l < q.r) {
        uint32_t tx, ty;
        if (q.s_log2) {  // base-s digits are bit fields
          tx = (x >> (l * q.s_log2)) & (s - 1);
          ty = (y >> (l * q.s_log2)) & (s - 1);
        } else {
          const uint32_t p = s_pw[l];
          tx = (x / p) % s;
          ty = (y / p) % s;
        }
        const int h = s_h[ty * s + tx];
        hole |= h < 0;
        a |= (uint32_t)(h < 0 ? 0 : h) << (8 * i);
      }
    }
    return a;
  };

  for (uint64_t base = warp0 * 16; base < count; base += nwarps * 16) {
    const uint64_t r0 = base + g, r1 = base + g + 8;
    const uint32_t x0 = r0 < count ? xi[r0] : 0u, y0 = r0 < count ? yi[r0] : 0u;
    const uint32_t x1 = r1 < count ? xi[r1] : 0u, y1 = r1 < count ? yi[r1] : 0u;
    bool h0 = (uint64_t)x0 >= q.n || (uint64_t)y0 >= q.n, h1 = (uint64_t)x1 >= q.n || (uint64_t)y1 >= q.n;
    // A fragment (16 x 32, row-major): a0 row g cols 4t.., a1 row g+8 cols 4t.., a2/a3 cols 16+4t..
    const uint32_t a0 = levels(x0, y0, 4 * t, h0), a1 = levels(x1, y1, 4 * t, h1);
    const uint32_t a2 = levels(x0, y0, 16 + 4 * t, h0), a3 = levels(x1, y1, 16 + 4 * t, h1);
    uint32_t d0, d1, d2, d3;
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%10, %10, %10, %10};"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0u));
    // D row g: columns (weight bytes) 2t, 2t+1 in d0, d1; row g+8 in d2, d3
    uint64_t v0 = ((uint64_t)d0 << (16 * t)) + ((uint64_t)d1 << (16 * t + 8));
    uint64_t v1 = ((uint64_t)d2 << (16 * t)) + ((uint64_t)d3 << (16 * t + 8));
    uint32_t hf = (h0 ? 1u : 0u) | (h1 ? 2u : 0u);
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      v0 += __shfl_xor_sync(0xFFFFFFFFu, v0, o);
      v1 += __shfl_xor_sync(0xFFFFFFFFu, v1, o);
      hf |= __shfl_xor_sync(0xFFFFFFFFu, hf, o);
    }
    if (t == 0) {
      if (r0 < count) om[r0] = (hf & 1u) ? kNoneU64 : v0;
      if (r1 < count) om[r1] = (hf & 2u) ? kNoneU64 : v1;
    }
  }
}

cudaError_t launch_map_nu_mma(const MmaNuParams& q, const uint32_t* x, const uint32_t* y, uint64_t* om,
                              uint64_t count, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  uint64_t blocks = (count + 127) / 128;  // 8 warps x 16 coordinates per CTA pass
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  k_map_nu_mma<<<(unsigned)blocks, 256, 0, st>>>(q, x, y, om, count);
  return cudaGetLastError();
}

}  // namespace sqz
