// sqz_engines.cu — the paper's comparison engines, rebuilt for sm_100a.
//
//  λ(ω) engine ("Compact grid and expanded fractal"): one thread per compact cell Ω
//    computes λ(Ω) and updates the cell in place of the EXPANDED bounding-box grid
//    (the BB layout of squeeze_bb_*: n x n bytes, 2 = hole).  No ν is needed: neighbours are
//    read by expanded address, holes and the border are skipped.
//  Block-level Squeeze: blocks of ρ x ρ = s^m x s^m expanded cells, one per
//    compact block index b in [0, k^(r-m)); block b stores the ρ x ρ micro-embedding of its
//    level-m sub-fractal (2 = hole).  The CTA computes λ_{r-m}(b) once and ν_{r-m} of the 8
//    neighbouring block coordinates once ("block-level Squeeze ... requiring less
//    operations, allowing thread cooperation"), then every thread updates one micro cell.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "sqz_bits.cuh"

namespace sqz {

__device__ __forceinline__ uint32_t rule_of(uint32_t alive, uint32_t count, uint32_t birth, uint32_t survive) {
  return ((alive ? survive : birth) >> count) & 1u;
}

// ------------------------------------------------------------------------------------ λ(ω) engine
__global__ void k_lambda_engine(LevelMaps gm, const uint8_t* __restrict__ cur, uint8_t* __restrict__ next,
                                uint32_t birth, uint32_t survive) {
  extern __shared__ uint32_t s_lut[];
  // stage the λ lookup tables in shared memory
  LevelMaps m = gm;
  {
    uint32_t n0 = gm.n_lam_full, n1 = gm.n_lam_tail;
    for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) s_lut[i] = gm.lam_full[i];
    for (uint32_t i = threadIdx.x; i < n1; i += blockDim.x) s_lut[n0 + i] = gm.lam_tail[i];
    m.lam_full = s_lut;
    m.lam_tail = s_lut + n0;
    __syncthreads();
  }
  const int64_t n = (int64_t)m.n;
  for (uint64_t om = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; om < m.cells;
       om += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x, y;
    lambda_level(m, om, x, y);
    uint32_t count = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t xx = (int64_t)x + moore_dx(i), yy = (int64_t)y + moore_dy(i);
      if (xx >= 0 && yy >= 0 && xx < n && yy < n) count += __ldg(cur + (uint64_t)yy * n + xx) == 1u;
    }
    const uint64_t at = (uint64_t)y * n + x;
    next[at] = (uint8_t)rule_of(__ldg(cur + at) == 1u, count, birth, survive);
  }
}

cudaError_t launch_lambda_engine(const LevelMaps& m, const uint8_t* cur, uint8_t* next, uint32_t birth,
                                 uint32_t survive, cudaStream_t st) {
  const size_t sm = (size_t)(m.n_lam_full + m.n_lam_tail) * 4;
  cudaError_t e = cudaSuccess;
  if (sm > 48 * 1024) e = cudaFuncSetAttribute((const void*)k_lambda_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (m.cells + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  k_lambda_engine<<<(unsigned)(blocks ? blocks : 1), 256, sm, st>>>(m, cur, next, birth, survive);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ block-level Squeeze
struct BlockParams {
  LevelMaps coarse;        // maps at level r_b = r - m (block coordinates)
  uint32_t rho;            // s^m
  uint32_t birth, survive;
  const uint8_t* micro;    // rho x rho micro-fractal mask (1 member, 0 hole)
};

// One CTA per group of blocks: threads [g*rho^2, (g+1)*rho^2) update block (base + g).
__global__ void k_block_step(BlockParams bp, const uint8_t* __restrict__ cur, uint8_t* __restrict__ next,
                             uint64_t nblocks, uint32_t blocks_per_cta) {
  __shared__ uint64_t s_nb[32][9];  // per block in the CTA: base offset of itself and its 8 neighbours (or ~0)
  const uint32_t rho = bp.rho, rr = rho * rho;
  const uint32_t g = threadIdx.x / rr, cell = threadIdx.x - g * rr;
  for (uint64_t base = (uint64_t)blockIdx.x * blocks_per_cta; base < nblocks;
       base += (uint64_t)gridDim.x * blocks_per_cta) {
    // block coordinates once per block (λ), neighbour blocks once per block (ν)
    for (uint32_t k = threadIdx.x; k < blocks_per_cta * 9; k += blockDim.x) {
      const uint32_t gi = k / 9, d = k - gi * 9;
      const uint64_t b = base + gi;
      uint64_t v = ~0ull;
      if (b < nblocks) {
        uint32_t X, Y;
        lambda_level(bp.coarse, b, X, Y);
        const int dx = (int)(d % 3) - 1, dy = (int)(d / 3) - 1;
        const uint64_t nb = (dx == 0 && dy == 0) ? b : nu_level(bp.coarse, (int64_t)X + dx, (int64_t)Y + dy);
        if (nb != kNoneU64) v = nb * rr;
      }
      s_nb[gi][d] = v;
    }
    __syncthreads();
    const uint64_t b = base + g;
    if (g < blocks_per_cta && b < nblocks) {
      const uint32_t u = cell % rho, w = cell / rho;
      const uint64_t at = b * rr + cell;
      const uint32_t self = __ldg(cur + at);
      uint8_t out = 2;
      if (self != 2u) {
        uint32_t count = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int xx = (int)u + moore_dx(i), yy = (int)w + moore_dy(i);
          const int bx = xx < 0 ? 0 : (xx >= (int)rho ? 2 : 1), by = yy < 0 ? 0 : (yy >= (int)rho ? 2 : 1);
          const uint64_t nbase = s_nb[g][by * 3 + bx];
          if (nbase == ~0ull) continue;
          xx -= (bx - 1) * (int)rho;
          yy -= (by - 1) * (int)rho;
          count += __ldg(cur + nbase + (uint32_t)yy * rho + (uint32_t)xx) == 1u;
        }
        out = (uint8_t)rule_of(self == 1u, count, bp.birth, bp.survive);
      }
      next[at] = out;
    }
    __syncthreads();
  }
}

// Seed: micro cell of block b = expanded (X*rho + u, Y*rho + w); holes of the micro mask = 2.
__global__ void k_block_seed(BlockParams bp, uint8_t* __restrict__ blocks, uint64_t nblocks, uint64_t mseed,
                             uint64_t q) {
  const uint32_t rr = bp.rho * bp.rho;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nblocks * rr;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = i / rr;
    const uint32_t cell = (uint32_t)(i - b * rr);
    uint8_t v = 2;
    if (bp.micro[cell]) {
      uint32_t X, Y;
      lambda_level(bp.coarse, b, X, Y);
      const uint32_t x = X * bp.rho + cell % bp.rho, y = Y * bp.rho + cell / bp.rho;
      uint64_t z = ((((uint64_t)x) << 32) | y) ^ mseed;
      z ^= z >> 30;
      z *= 0xBF58476D1CE4E5B9ull;
      z ^= z >> 27;
      z *= 0x94D049BB133111EBull;
      z ^= z >> 31;
      v = (z >> 32) < q ? 1 : 0;
    }
    blocks[i] = v;
  }
}

cudaError_t launch_block_step(const LevelMaps& coarse, uint32_t rho, const uint8_t* micro, uint32_t birth,
                              uint32_t survive, const uint8_t* cur, uint8_t* next, cudaStream_t st) {
  BlockParams bp{coarse, rho, birth, survive, micro};
  const uint32_t rr = rho * rho;
  const uint32_t per = rr >= 256 ? 1u : std::min(32u, 256u / rr);
  const uint32_t threads = per * rr;
  const uint64_t nblocks = coarse.cells;
  uint64_t grid = (nblocks + per - 1) / per;
  if (grid > 148ull * 32) grid = 148ull * 32;
  k_block_step<<<(unsigned)(grid ? grid : 1), threads, 0, st>>>(bp, cur, next, nblocks, per);
  return cudaGetLastError();
}

cudaError_t launch_block_seed(const LevelMaps& coarse, uint32_t rho, const uint8_t* micro, uint8_t* blocks,
                              uint64_t seed, uint64_t q, cudaStream_t st) {
  BlockParams bp{coarse, rho, 0, 0, micro};
  uint64_t z = seed;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  const uint64_t total = coarse.cells * rho * rho;
  uint64_t grid = (total + 255) / 256;
  if (grid > 148ull * 32) grid = 148ull * 32;
  k_block_seed<<<(unsigned)(grid ? grid : 1), 256, 0, st>>>(bp, blocks, coarse.cells, z, q);
  return cudaGetLastError();
}

}  // namespace sqz
