// sqz_heat.cu — second workload (reading D16): explicit heat
// diffusion on the compact form of an NBB fractal,
//
//     u'(Ω) = u(Ω) + α Σ_{n ∈ N(Ω)} (u(n) − u(Ω)),   N(Ω) = member Moore neighbours,
//
// with the automaton's neighbour machinery ("PDE solvers ... rely on accessing
// neighboring cells").  float32 state, one value per compact cell.
//
// Layout (include/squeeze.h): tile-padded floats, local tile t at float offset t·Kf,
// Kf = round_up(K, 4) (16-byte aligned tiles; padding floats are 0).
//
// Tables (host, from the level-g tile tables): every cell j has 8 neighbour slots (the first D read)
// holding byte offsets relative to its tile's shared-memory slot — a local cell j', the cell
// ITSELF for an absent neighbour (a zero term), or a remote PAIR p at float Kf + p.  Pairs are
// per (own cell, neighbour) so that a pair whose neighbour tile does not exist (the fractal's
// edge) can hold the own value: the insulated boundary costs no degree bookkeeping.  With the
// absent slots as the cell itself, Σ_n (u_n − u) = Σ_{slots} u_s − D·u for the fixed slot count D.
//
// Kernel: CTA = 8 warps, work unit = 8 consecutive tiles, bulk-copied into a stage with the
// tiles' adjacency words; warp m fills tile m's pair slots (neighbour tile from the adjacency
// table — coarse λ + ν at init, P:189 at tile level); after one CTA barrier warp w updates its
// static j-blocks (neighbour slots held in registers for the whole launch) in all 8 tiles, with
// coalesced stores straight to HBM.  HBM-bound: 8 B per cell per step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_bits.cuh"
#include "sqz_heat.cuh"

namespace sqz {

constexpr uint32_t kHeatTiles = 8;  // tiles per work unit = warps per CTA

__host__ __device__ inline uint32_t heat_cf(const HeatParams& h) { return (h.Kf + h.P + 3) & ~3u; }

struct HeatSmem {
  float* U0;      // stages x kHeatTiles x Cf floats ([Kf state | P pairs] per tile)
  uint32_t* A0;   // stages x ndirs x kHeatTiles adjacency words
  uint64_t* bar;  // stages
  uint32_t sw, aw;
};

__host__ __device__ inline size_t heat_layout(const HeatParams& h, const TileParams& p, uint8_t* base, HeatSmem* s) {
  const size_t sw = (size_t)kHeatTiles * heat_cf(h), aw = (size_t)p.ndirs * kHeatTiles;
  size_t off = 0;
  if (s) {
    s->U0 = (float*)base;
    s->sw = (uint32_t)sw;
    s->aw = (uint32_t)aw;
  }
  off += (size_t)h.stages * sw * 4;
  if (s) s->A0 = (uint32_t*)(base + off);
  off += align16((size_t)h.stages * (aw ? aw : 1) * 4);
  if (s) s->bar = (uint64_t*)(base + off);
  off += (size_t)h.stages * 8;
  return align16(off);
}

size_t heat_smem_bytes(const HeatParams& h, const TileParams& p) { return heat_layout(h, p, nullptr, nullptr); }

__device__ __forceinline__ void heat_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One thread: the unit's nt tiles (Kf floats each) and adjacency words -> stage s.
__device__ __forceinline__ void heat_load(const HeatParams& h, const TileParams& p, const HeatSmem& S, uint64_t unit,
                                          uint32_t s, const float* __restrict__ cur) {
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  const uint64_t t0 = unit * kHeatTiles;
  const uint32_t nt = (uint32_t)min((uint64_t)kHeatTiles, ntl - t0);
  const uint32_t tb = h.Kf * 4, ab = kHeatTiles * 4;
  uint64_t* bar = &S.bar[s];
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(tb * nt + ab * p.ndirs)
               : "memory");
  const uint32_t u = smem_u32(S.U0 + (size_t)s * S.sw), a = smem_u32(S.A0 + (size_t)s * S.aw);
  const uint32_t cf = heat_cf(h);
  for (uint32_t m = 0; m < nt; ++m) heat_g2s(u + m * cf * 4, cur + (t0 + m) * h.Kf, tb, bar);
  for (uint32_t d = 0; d < p.ndirs; ++d) heat_g2s(a + d * ab, p.adj + d * p.adj_stride + t0, ab, bar);
}

// D: neighbour slots read per cell (5 for the Sierpinski triangle, else 8).  RB: j-blocks per
// warp with register-resident slots (block jb = warp + i * 8, all 8 tiles of a unit); later
// blocks read their slots through L1.
template <int D, int RB>
__global__ void __launch_bounds__(256, 3) k_heat_step(HeatParams h, TileParams p, const float* __restrict__ cur,
                                                      float* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  HeatSmem S;
  heat_layout(h, p, smem_raw, &S);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t K = (uint32_t)p.K, Kf = h.Kf, cf = heat_cf(h), NS = h.stages;
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  const uint64_t nunits = (ntl + kHeatTiles - 1) / kHeatTiles;
  const bool issuer = threadIdx.x == 0;
  const float alpha = h.alpha;

  uint32_t off[RB][D];  // byte offsets of this lane's neighbour slots (relative to a tile slot)
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t j = ((uint32_t)warp + (uint32_t)i * kHeatTiles) * 32 + lane;
    const uint4 row = j < K ? __ldg(reinterpret_cast<const uint4*>(h.nbr) + j) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {row.x, row.y, row.z, row.w};
#pragma unroll
    for (int k = 0; k < D; ++k) off[i][k] = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
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

  // pair slots of tile `warp` of a unit: the neighbour cell's value, or the own cell's (absent tile)
  auto fill_pairs = [&](uint64_t u, uint32_t st) {
    const uint64_t t0 = u * kHeatTiles;
    const uint32_t nt = (uint32_t)min((uint64_t)kHeatTiles, ntl - t0);
    if ((uint32_t)warp >= nt) return;
    float* U = S.U0 + (size_t)st * S.sw;
    const uint32_t* A = S.A0 + (size_t)st * S.aw;
    float* T = U + (size_t)warp * cf;
    for (uint32_t q = lane; q < h.P; q += 32) {
      const uint32_t pr = __ldg(h.pairs + q);  // own cell j | link direction << 16
      const uint32_t j = pr & 0xFFFFu, d = pr >> 16;
      const uint32_t j2 = __ldg(h.pair_j2 + q);
      const uint32_t a1 = A[d * kHeatTiles + warp];
      float v = T[j];
      if (a1 != 0) {
        const uint64_t tn = (uint64_t)(a1 - 1) - p.tile_lo;
        v = (tn >= t0 && tn < t0 + nt) ? U[(size_t)(tn - t0) * cf + j2] : __ldg(cur + tn * Kf + j2);
      }
      T[Kf + q] = v;
    }
  };
  // One CTA barrier per unit: it publishes the NEXT unit's pair slots (filled after this unit's
  // cells) and frees this unit's stage for the refill.
  uint32_t s = 0, ph = 0;
  mbar_wait(&S.bar[0], 0);
  ph = 1;
  fill_pairs(unit, 0);
  __syncthreads();
  for (; unit < nunits; unit += G, s = (s + 1 == NS) ? 0 : s + 1) {
    const uint64_t t0 = unit * kHeatTiles;  // local index of the unit's first tile
    const uint32_t nt = (uint32_t)min((uint64_t)kHeatTiles, ntl - t0);
    const float* U = S.U0 + (size_t)s * S.sw;

    // warp = j-block across the unit's tiles; lane = cell
    auto cellblock = [&](uint32_t j, const uint32_t* o) {
      for (uint32_t m = 0; m < nt; ++m) {
        const uint8_t* T = reinterpret_cast<const uint8_t*>(U + (size_t)m * cf);
        float nv = 0.0f;
        if (j < K) {
          float x[D];
#pragma unroll
          for (int k = 0; k < D; ++k) x[k] = *reinterpret_cast<const float*>(T + o[k]);
          // pairwise sum (its rounding is within the sequential-order bound of oracle/heat.py)
          float sum = (x[0] + x[1]) + (x[2] + x[3]);
          if (D == 5) sum += x[4 % D];
          if (D == 8) sum += (x[4 % D] + x[5 % D]) + (x[6 % D] + x[7 % D]);
          const float u = reinterpret_cast<const float*>(T)[j];
          nv = fmaf(alpha, sum - (float)D * u, u);
        }
        next[(t0 + m) * Kf + j] = nv;  // padding floats K..Kf-1 are written 0
      }
    };
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const uint32_t j = ((uint32_t)warp + (uint32_t)i * kHeatTiles) * 32 + lane;
      if (j - lane < Kf && j < Kf) cellblock(j, off[i]);
    }
    for (uint32_t j = ((uint32_t)warp + (uint32_t)RB * kHeatTiles) * 32 + lane; j < Kf; j += kHeatTiles * 32) {
      const uint4 row = j < K ? __ldg(reinterpret_cast<const uint4*>(h.nbr) + j) : make_uint4(0, 0, 0, 0);
      const uint32_t w[4] = {row.x, row.y, row.z, row.w};
      uint32_t o[D];
#pragma unroll
      for (int k = 0; k < D; ++k) o[k] = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      cellblock(j, o);
    }
    if (unit + G < nunits) {  // the next unit's stage was issued NS - 1 units ago
      const uint32_t s1 = (s + 1 == NS) ? 0 : s + 1;
      mbar_wait(&S.bar[s1], (ph >> s1) & 1);
      ph ^= 1u << s1;
      fill_pairs(unit + G, s1);
    }
    __syncthreads();  // next unit's pairs in place; every warp is done with stage s
    if (issuer && unit + NS * G < nunits) {
      fence_proxy_async();
      heat_load(h, p, S, unit + NS * G, s, cur);
    }
  }
}

// Initial field: u(Ω) = heat_value at λ(Ω) (D16), padding floats 0.
__global__ void k_heat_seed(LevelMaps gm, uint64_t tile_lo, uint64_t ntiles, uint32_t K, uint32_t Kf, float* u,
                            uint64_t mseed) {
  const uint64_t n = ntiles * Kf;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / Kf;
    const uint32_t j = (uint32_t)(i - t * Kf);
    float v = 0.0f;
    if (j < K) {
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

// Σu in float64 (padding floats are 0).
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

using HeatFn = void (*)(HeatParams, TileParams, const float*, float*);

static HeatFn pick_heat(const TileParams& p) {
  return p.dmax <= 5 ? k_heat_step<5, 3> : k_heat_step<8, 2>;
}

cudaError_t heat_prepare(const HeatParams& h, const TileParams& p, int* occupancy) {
  HeatFn fn = pick_heat(p);
  const size_t smem = heat_smem_bytes(h, p);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 32 * kHeatTiles, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t launch_heat_step(const HeatParams& h, const TileParams& p, const float* cur, float* next, int grid,
                             cudaStream_t st) {
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  if (ntl == 0) return cudaSuccess;
  const uint64_t units = (ntl + kHeatTiles - 1) / kHeatTiles;
  const int g = (int)(units < (uint64_t)grid ? units : (uint64_t)grid);
  pick_heat(p)<<<g, 32 * kHeatTiles, heat_smem_bytes(h, p), st>>>(h, p, cur, next);
  return cudaGetLastError();
}

cudaError_t launch_heat_seed(const LevelMaps& full, const TileParams& p, uint32_t Kf, float* u, uint64_t seed,
                             cudaStream_t st) {
  const uint64_t ntl = p.tile_hi - p.tile_lo;
  if (ntl == 0) return cudaSuccess;
  uint64_t z = seed;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  uint64_t blocks = (ntl * Kf + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_heat_seed<<<(unsigned)blocks, 256, 0, st>>>(full, p.tile_lo, ntl, (uint32_t)p.K, Kf, u, z);
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
