// sqz_heat.cu — second workload (reading D16): explicit heat
// diffusion on the compact form of an NBB fractal,
//
//     u'(Ω) = u(Ω) + α Σ_{n ∈ N(Ω)} (u(n) − u(Ω)),   N(Ω) = member Moore neighbours,
//
// with the automaton's neighbour machinery ("PDE solvers ... rely on accessing
// neighboring cells").  float32 state, one value per compact cell.
//
// Layout (include/squeeze.h): the shard's level-g tiles in chunks of kHeatLanes = 4; chunk c
// holds K float4 words, word j = cell j of tiles 4c..4c+3 (lane l = tile 4c + l).  As in the
// packed automaton, one 128-bit shared-memory load fetches a neighbour for 4 cells.
//
// Tables (host, from the level-g tile tables): every cell j has 8 neighbour slots (the first D
// read) — a local cell j', the cell ITSELF for an absent neighbour (a zero term), or a remote
// PAIR p at word K + p of the chunk's slot.  Pairs are per (own cell, neighbour) so that a
// pair whose neighbour tile does not exist (the fractal's edge) can hold the own value: the
// insulated boundary costs no degree bookkeeping, and Σ_n (u_n − u) = Σ_{slots} u_s − D·u.
//
// Kernel: CTA = 8 warps; unit = kHeatChunks chunks bulk-copied into a stage with the unit's
// adjacency words (coarse λ + ν per tile at init, P:189 at tile level).  The pairs of the next
// unit are filled while this one is computed; warp w updates its static j-blocks (neighbour
// slots in registers for the whole launch) in every chunk of the unit, one coalesced 512-byte
// float4 store per warp straight to HBM.  One CTA barrier per unit.  HBM-bound: 8 B per cell.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_bits.cuh"
#include "sqz_heat.cuh"

namespace sqz {

constexpr uint32_t kHeatLanes = 4;   // tiles per chunk (float4 lanes)
constexpr uint32_t kHeatChunks = 2;  // chunks per work unit
constexpr uint32_t kHeatUnitTiles = kHeatLanes * kHeatChunks;

__host__ __device__ inline uint32_t heat_cw(const HeatParams& h) { return h.K + h.P; }  // float4 words per chunk slot

struct HeatSmem {
  float4* U0;     // stages x kHeatChunks x cw float4 ([K state | P pairs] per chunk)
  uint32_t* A0;   // stages x ndirs x kHeatUnitTiles adjacency words
  uint64_t* bar;  // stages
  uint32_t sw, aw;
};

__host__ __device__ inline size_t heat_layout(const HeatParams& h, const TileParams& p, uint8_t* base, HeatSmem* s) {
  const size_t sw = (size_t)kHeatChunks * heat_cw(h), aw = (size_t)p.ndirs * kHeatUnitTiles;
  size_t off = 0;
  if (s) {
    s->U0 = (float4*)base;
    s->sw = (uint32_t)sw;
    s->aw = (uint32_t)aw;
  }
  off += (size_t)h.stages * sw * 16;
  if (s) s->A0 = (uint32_t*)(base + off);
  off += align16((size_t)h.stages * (aw ? aw : 1) * 4);
  if (s) s->bar = (uint64_t*)(base + off);
  off += (size_t)h.stages * 8;
  return align16(off);
}

size_t heat_smem_bytes(const HeatParams& h, const TileParams& p) { return heat_layout(h, p, nullptr, nullptr); }

__host__ __device__ inline uint64_t heat_chunks(const TileParams& p) {
  return (p.tile_hi - p.tile_lo + kHeatLanes - 1) / kHeatLanes;
}

__device__ __forceinline__ void heat_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One thread: the unit's nc chunks (K float4 each) and its adjacency words -> stage s.
// (Adjacency rows are padded to whole 128-tile chunks on the host: every copy stays in bounds.)
__device__ __forceinline__ void heat_load(const HeatParams& h, const TileParams& p, const HeatSmem& S, uint64_t unit,
                                          uint32_t s, const float4* __restrict__ cur) {
  const uint64_t c0 = unit * kHeatChunks;
  const uint32_t nc = (uint32_t)min((uint64_t)kHeatChunks, heat_chunks(p) - c0);
  const uint32_t cb = h.K * 16, ab = kHeatUnitTiles * 4;
  uint64_t* bar = &S.bar[s];
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(cb * nc + ab * p.ndirs)
               : "memory");
  const uint32_t u = smem_u32(S.U0 + (size_t)s * S.sw), a = smem_u32(S.A0 + (size_t)s * S.aw);
  const uint32_t cw = heat_cw(h);
  for (uint32_t m = 0; m < nc; ++m) heat_g2s(u + m * cw * 16, cur + (c0 + m) * h.K, cb, bar);
  for (uint32_t d = 0; d < p.ndirs; ++d) heat_g2s(a + d * ab, p.adj + d * p.adj_stride + c0 * kHeatLanes, ab, bar);
}

template <int D>
__device__ __forceinline__ float heat_update(const float* x, float u, float alpha) {
  // pairwise sum (its rounding stays within the sequential-order bound of oracle/heat.py)
  float sum = (x[0] + x[1]) + (x[2] + x[3]);
  if (D == 5) sum += x[4 % D];
  if (D == 8) sum += (x[4 % D] + x[5 % D]) + (x[6 % D] + x[7 % D]);
  return fmaf(alpha, sum - (float)D * u, u);
}

// D: neighbour slots read per cell (5 for the Sierpinski triangle, else 8).  RB: j-blocks per
// warp with register-resident slots (block jb = warp + 8 i); later blocks read theirs via L1.
template <int D, int RB>
__global__ void __launch_bounds__(256, 3) k_heat_step(HeatParams h, TileParams p, const float4* __restrict__ cur,
                                                      float4* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  HeatSmem S;
  heat_layout(h, p, smem_raw, &S);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t K = h.K, cw = heat_cw(h), NS = h.stages;
  const uint64_t nch = heat_chunks(p);
  const uint64_t nunits = (nch + kHeatChunks - 1) / kHeatChunks;
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  const bool issuer = threadIdx.x == 0;
  const float alpha = h.alpha;

  uint32_t off[RB][D];  // byte offsets of this lane's neighbour words in a chunk slot
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t j = ((uint32_t)warp + (uint32_t)(i * nwarps)) * 32 + lane;
    const uint4 row = j < K ? __ldg(reinterpret_cast<const uint4*>(h.nbr) + j) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {row.x, row.y, row.z, row.w};
#pragma unroll
    for (int k = 0; k < D; ++k) off[i][k] = ((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) * 16;
  }

  if (issuer) {
    for (uint32_t s = 0; s < NS; ++s) mbar_init(&S.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t unit = blockIdx.x;
  const uint64_t G = gridDim.x;
  if (issuer)
    for (uint32_t s = 0; s < NS && unit + s * G < nunits; ++s) heat_load(h, p, S, unit + s * G, s, cur);

  // pair slots of a unit, item i = (pair q, tile of the unit): the neighbour cell's value, or
  // the own cell's when the neighbour tile does not exist.  pair_value reads it (from the
  // stage, or from HBM for a neighbour tile outside the unit) without storing it, so the
  // next unit's values can be in flight while this unit's cells are computed.
  auto pair_value = [&](uint64_t t0, const float* U, const uint32_t* A, uint32_t i) -> float {
    const uint32_t q = i / kHeatUnitTiles, tu = i % kHeatUnitTiles;  // pair, tile of the unit
    const uint32_t m = tu / kHeatLanes, l = tu % kHeatLanes;
    const uint32_t pr = __ldg(h.pairs + q);  // own cell j | link direction << 16
    const uint32_t j = pr & 0xFFFFu, d = pr >> 16;
    const uint32_t a1 = A[d * kHeatUnitTiles + tu];
    if (a1 == 0 || t0 + tu >= ntl) return U[((size_t)m * cw + j) * 4 + l];
    const uint32_t j2 = __ldg(h.pair_j2 + q);
    const uint64_t tn = (uint64_t)(a1 - 1) - p.tile_lo;  // local neighbour tile
    const uint64_t rel = tn - t0;
    return rel < kHeatUnitTiles
               ? U[((size_t)(rel / kHeatLanes) * cw + j2) * 4 + rel % kHeatLanes]
               : __ldg(reinterpret_cast<const float*>(cur) + ((tn / kHeatLanes) * K + j2) * 4 + tn % kHeatLanes);
  };
  auto pair_slot = [&](float* U, uint32_t i) -> float& {
    const uint32_t q = i / kHeatUnitTiles, tu = i % kHeatUnitTiles;
    return U[((size_t)(tu / kHeatLanes) * cw + K + q) * 4 + tu % kHeatLanes];
  };
  const uint32_t npi = h.P * kHeatUnitTiles;  // pair items per unit

  uint32_t s = 0, ph = 1;
  mbar_wait(&S.bar[0], 0);
  {
    float* U = reinterpret_cast<float*>(S.U0);
    for (uint32_t i = threadIdx.x; i < npi; i += blockDim.x) pair_slot(U, i) = pair_value(unit * kHeatUnitTiles, U, S.A0, i);
  }
  __syncthreads();
  for (; unit < nunits; unit += G, s = (s + 1 == NS) ? 0 : s + 1) {
    const uint64_t c0 = unit * kHeatChunks;
    const uint32_t nc = (uint32_t)min((uint64_t)kHeatChunks, nch - c0);
    const uint32_t us = smem_u32(S.U0 + (size_t)s * S.sw);
    // the next unit's first two pair items of this thread, gathered before this unit's cells
    const bool has_next = unit + G < nunits;
    const uint32_t s1 = (s + 1 == NS) ? 0 : s + 1;
    float* U1 = reinterpret_cast<float*>(S.U0 + (size_t)s1 * S.sw);
    const uint32_t* A1 = S.A0 + (size_t)s1 * S.aw;
    float pv0 = 0.0f, pv1 = 0.0f;
    if (has_next) {  // its stage was issued NS - 1 units ago
      mbar_wait(&S.bar[s1], (ph >> s1) & 1);
      ph ^= 1u << s1;
      const uint64_t t1 = (unit + G) * kHeatUnitTiles;
      if (threadIdx.x < npi) pv0 = pair_value(t1, U1, A1, threadIdx.x);
      if (threadIdx.x + blockDim.x < npi) pv1 = pair_value(t1, U1, A1, threadIdx.x + blockDim.x);
    }
    auto block = [&](uint32_t j, const uint32_t* o) {
      if (j >= K) return;
      for (uint32_t m = 0; m < nc; ++m) {
        const uint32_t base = us + m * cw * 16;
        float x0[D], x1[D], x2[D], x3[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const uint4 v = lds128(base + o[k]);
          x0[k] = __uint_as_float(v.x);
          x1[k] = __uint_as_float(v.y);
          x2[k] = __uint_as_float(v.z);
          x3[k] = __uint_as_float(v.w);
        }
        const uint4 uu = lds128(base + j * 16);
        float4 nv;
        nv.x = heat_update<D>(x0, __uint_as_float(uu.x), alpha);
        nv.y = heat_update<D>(x1, __uint_as_float(uu.y), alpha);
        nv.z = heat_update<D>(x2, __uint_as_float(uu.z), alpha);
        nv.w = heat_update<D>(x3, __uint_as_float(uu.w), alpha);
        next[(c0 + m) * K + j] = nv;  // lanes of tiles past the shard end stay 0 (inputs 0)
      }
    };
#pragma unroll
    for (int i = 0; i < RB; ++i) block(((uint32_t)warp + (uint32_t)(i * nwarps)) * 32 + lane, off[i]);
    for (uint32_t j = ((uint32_t)warp + (uint32_t)(RB * nwarps)) * 32 + lane; j - lane < K; j += nwarps * 32) {
      const uint4 row = j < K ? __ldg(reinterpret_cast<const uint4*>(h.nbr) + j) : make_uint4(0, 0, 0, 0);
      const uint32_t w[4] = {row.x, row.y, row.z, row.w};
      uint32_t o[D];
#pragma unroll
      for (int k = 0; k < D; ++k) o[k] = ((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) * 16;
      block(j, o);
    }
    if (has_next) {
      const uint64_t t1 = (unit + G) * kHeatUnitTiles;
      if (threadIdx.x < npi) pair_slot(U1, threadIdx.x) = pv0;
      if (threadIdx.x + blockDim.x < npi) pair_slot(U1, threadIdx.x + blockDim.x) = pv1;
      for (uint32_t i = threadIdx.x + 2 * blockDim.x; i < npi; i += blockDim.x)
        pair_slot(U1, i) = pair_value(t1, U1, A1, i);
    }
    __syncthreads();  // next unit's pairs in place; every warp is done with stage s
    if (issuer && unit + NS * G < nunits) {
      fence_proxy_async();
      heat_load(h, p, S, unit + NS * G, s, cur);
    }
  }
}

// Initial field: u(Ω) = heat_value at λ(Ω) (D16); lanes of tiles past the shard end 0.
__global__ void k_heat_seed(LevelMaps gm, uint64_t tile_lo, uint64_t ntiles, uint32_t K, float* u, uint64_t mseed) {
  const uint64_t n = (ntiles + kHeatLanes - 1) / kHeatLanes * K * kHeatLanes;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = i / kHeatLanes, c = w / K;
    const uint32_t l = (uint32_t)(i % kHeatLanes), j = (uint32_t)(w - c * K);
    const uint64_t t = c * kHeatLanes + l;
    float v = 0.0f;
    if (t < ntiles) {
      uint32_t x, y;
      lambda_level(gm, (tile_lo + t) * K + j, x, y);
      uint64_t z = ((((uint64_t)x) << 32) | y) ^ mseed;
      z ^= z >> 30;
      z *= 0xBF58476D1CE4E5B9ull;
      z ^= z >> 27;
      z *= 0x94D049BB133111EBull;
      z ^= z >> 31;
      v = (float)(z >> 40) * (1.0f / 16777216.0f);  // 24 bits: exact in float32
    }
    u[i] = v;
  }
}

// Σu in float64 (lanes past the shard end are 0).
__global__ void k_heat_sum(const float* __restrict__ u, uint64_t n, double* out) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += (double)u[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (threadIdx.x == 0) atomicAdd(out, v);
  }
}

using HeatFn = void (*)(HeatParams, TileParams, const float4*, float4*);

static HeatFn pick_heat(const HeatParams& h, const TileParams& p) {
  const uint32_t nblk = (h.K + 31) / 32;
  if (p.dmax <= 5) return nblk <= 24 ? k_heat_step<5, 3> : k_heat_step<5, 5>;
  return nblk <= 16 ? k_heat_step<8, 2> : k_heat_step<8, 3>;
}

cudaError_t heat_prepare(const HeatParams& h, const TileParams& p, int* occupancy) {
  HeatFn fn = pick_heat(h, p);
  const size_t smem = heat_smem_bytes(h, p);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 256, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t launch_heat_step(const HeatParams& h, const TileParams& p, const float* cur, float* next, int grid,
                             cudaStream_t st) {
  const uint64_t nunits = (heat_chunks(p) + kHeatChunks - 1) / kHeatChunks;
  if (nunits == 0) return cudaSuccess;
  const int g = (int)(nunits < (uint64_t)grid ? nunits : (uint64_t)grid);
  pick_heat(h, p)<<<g, 256, heat_smem_bytes(h, p), st>>>(h, p, reinterpret_cast<const float4*>(cur),
                                                          reinterpret_cast<float4*>(next));
  return cudaGetLastError();
}

cudaError_t launch_heat_seed(const LevelMaps& full, const TileParams& p, float* u, uint64_t seed, cudaStream_t st) {
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  if (ntl == 0) return cudaSuccess;
  uint64_t z = seed;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  const uint64_t n = heat_chunks(p) * p.K * kHeatLanes;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_heat_seed<<<(unsigned)blocks, 256, 0, st>>>(full, p.tile_lo, ntl, (uint32_t)p.K, u, z);
  return cudaGetLastError();
}

cudaError_t launch_heat_sum(const float* u, uint64_t n, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148ull * 4) blocks = 148ull * 4;
  k_heat_sum<<<(unsigned)(blocks ? blocks : 1), 256, 0, st>>>(u, n, out);
  return cudaGetLastError();
}

}  // namespace sqz
