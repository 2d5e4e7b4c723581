// sqz_kernels.cu — sm_100a kernels of the Squeeze hot path (arXiv 2201.00613).
//
// Kernels:
//   k_map_lambda / k_map_nu   batched λ / ν with the multi-digit
//                             lookup tables staged in shared memory
//   k_seed                    initial state (reading D9) at (X, Y) = λ(Ω)
//   k_step_naive              the paper's per-thread step: 1 λ + 8 (membership, ν,
//                             gather) per cell — the literal comparison engine
//   k_step_tile               the product step: 32 level-g tiles per work
//                             unit, bit-sliced one tile per bit, one shared intra-tile
//                             neighbour table, per-tile coarse λ + ν only for the tile
//                             boundary links, TMA bulk copies in and out of shared memory
//   k_count_alive, k_halo_pack, BB baseline (k_bb_seed, k_bb_step, k_bb_to_compact)
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_device.cuh"
#include "sqz_kernels.cuh"

namespace sqz {

// ---------------------------------------------------------------------------------------
// common device helpers

__device__ __forceinline__ uint64_t seed_mix(uint64_t z) {
  // splitmix64 finaliser (reading D9; same generator as sqz_inputs.mix)
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ uint32_t seed_alive(uint32_t x, uint32_t y, uint64_t mseed, uint64_t q) {
  uint64_t h = seed_mix((((uint64_t)x) << 32 | y) ^ mseed);
  return (h >> 32) < q ? 1u : 0u;
}

// Copies a LevelMaps' four LUTs into shared memory and returns a view on them.
__device__ __forceinline__ LevelMaps stage_maps(const LevelMaps& g, uint32_t* smem) {
  LevelMaps m = g;
  uint32_t* p = smem;
  uint32_t n0 = g.n_lam_full, n1 = g.n_lam_tail, n2 = g.n_nu_full, n3 = g.n_nu_tail;
  for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) p[i] = g.lam_full[i];
  for (uint32_t i = threadIdx.x; i < n1; i += blockDim.x) p[n0 + i] = g.lam_tail[i];
  for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) p[n0 + n1 + i] = g.nu_full[i];
  for (uint32_t i = threadIdx.x; i < n3; i += blockDim.x) p[n0 + n1 + n2 + i] = g.nu_tail[i];
  m.lam_full = p;
  m.lam_tail = p + n0;
  m.nu_full = p + n0 + n1;
  m.nu_tail = p + n0 + n1 + n2;
  __syncthreads();
  return m;
}

__host__ __device__ inline size_t maps_smem_bytes(const LevelMaps& m) {
  return (size_t)(m.n_lam_full + m.n_lam_tail + m.n_nu_full + m.n_nu_tail) * sizeof(uint32_t);
}

__device__ __forceinline__ uint32_t rule_byte(uint32_t alive, uint32_t count, uint32_t birth, uint32_t survive) {
  return ((alive ? survive : birth) >> count) & 1u;
}

// ---------------------------------------------------------------------------------------
// batched maps

__global__ void k_map_lambda(LevelMaps gm, const uint64_t* __restrict__ om, uint32_t* __restrict__ xo,
                             uint32_t* __restrict__ yo, uint64_t count) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t w = om[i];
    uint32_t x = 0xFFFFFFFFu, y = 0xFFFFFFFFu;
    if (w < m.cells) lambda_level(m, w, x, y);
    xo[i] = x;
    yo[i] = y;
  }
}

__global__ void k_map_nu(LevelMaps gm, const uint32_t* __restrict__ xi, const uint32_t* __restrict__ yi,
                         uint64_t* __restrict__ om, uint64_t count) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    om[i] = nu_level(m, (int64_t)xi[i], (int64_t)yi[i]);
}

// ---------------------------------------------------------------------------------------
// seed: 4 cells per thread, one 32-bit store; bytes past the shard are zero padding

__global__ void k_seed(LevelMaps gm, PadLayout L, uint64_t words, uint32_t* __restrict__ state, uint64_t mseed,
                       uint64_t q) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint64_t off = w * 4 + b;
      const uint64_t tl = fdiv(L.divKp, off);
      const uint64_t j = off - tl * L.Kp;
      if (j < L.K) {
        uint32_t x, y;
        lambda_level(m, (L.tile_lo + tl) * L.K + j, x, y);
        v |= seed_alive(x, y, mseed, q) << (8 * b);
      }
    }
    state[w] = v;
  }
}

// ---------------------------------------------------------------------------------------
// literal per-cell step: one λ, eight (membership + ν), gather, rule

__global__ void k_step_naive(LevelMaps gm, const uint8_t* __restrict__ cur, uint32_t* __restrict__ next, uint64_t words,
                             uint32_t birth, uint32_t survive, HaloView halo) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  const PadLayout& L = halo.L;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t out = 0;
#pragma unroll 1
    for (int b = 0; b < 4; ++b) {
      const uint64_t off = w * 4 + b;
      const uint64_t tl = fdiv(L.divKp, off);
      const uint64_t j = off - tl * L.Kp;
      if (j >= L.K) continue;  // tile padding stays zero
      const uint64_t om = (L.tile_lo + tl) * L.K + j;
      uint32_t x, y;
      lambda_level(m, om, x, y);
      uint32_t count = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint64_t nb = nu_level(m, (int64_t)x + moore_dx(i), (int64_t)y + moore_dy(i));
        if (nb != kNoneU64) count += fetch_cell(cur, nb, halo);
      }
      out |= rule_byte(__ldg(cur + off), count, birth, survive) << (8 * b);
    }
    next[w] = out;
  }
}

// ---------------------------------------------------------------------------------------
// alive count, halo pack

__global__ void k_count_alive(const uint4* __restrict__ st, uint64_t n16, const uint8_t* __restrict__ tail,
                              uint32_t ntail, unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = st[i];
    uint32_t s = __dp4a(v.x, 0x01010101u, 0u);
    s = __dp4a(v.y, 0x01010101u, s);
    s = __dp4a(v.z, 0x01010101u, s);
    s = __dp4a(v.w, 0x01010101u, s);
    acc += s;
  }
  if (blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < ntail; i += blockDim.x) acc += tail[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  __shared__ unsigned long long red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (threadIdx.x == 0) atomicAdd(out, v);
  }
}

// peer_recv[peer[i]][pos[i]] = cur[off_i]: the halo of a state written into the peers' buffers.
__global__ void k_halo_peer_push(const uint8_t* __restrict__ cur, const uint64_t* __restrict__ offs,
                                 const uint32_t* __restrict__ peer, const uint64_t* __restrict__ pos, uint64_t n,
                                 uint8_t* const* __restrict__ peer_recv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    peer_recv[peer[i]][pos[i]] = cur[offs[i]];
  __threadfence_system();
}

__global__ void k_halo_pack(const uint8_t* __restrict__ cur, const uint64_t* __restrict__ offs, uint64_t n,
                            uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = cur[offs[i]];
}

// ---------------------------------------------------------------------------------------
// BB baseline: expanded n x n grid, 0 dead / 1 alive / 2 hole ("BB")

__global__ void k_bb_seed(LevelMaps gm, uint8_t* __restrict__ grid, uint64_t n, uint64_t mseed, uint64_t q) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  uint64_t total = n * n;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t y = i / n, x = i - y * n;
    uint64_t om = nu_level(m, (int64_t)x, (int64_t)y);
    grid[i] = (om == kNoneU64) ? 2 : (uint8_t)seed_alive((uint32_t)x, (uint32_t)y, mseed, q);
  }
}


// generic per-cell BB step (n % 32 != 0, e.g. s = 3 fractals); powers of two take sqz_bb.cu
__global__ void k_bb_step1(const uint8_t* __restrict__ cur, uint8_t* __restrict__ next, uint64_t n, uint32_t birth,
                           uint32_t survive) {
  uint64_t total = n * n;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t y = (int64_t)(i / n), x = (int64_t)(i - (uint64_t)y * n);
    uint32_t v = cur[i];
    if (v == 2u) {
      next[i] = 2;
      continue;
    }
    uint32_t c = 0;
    for (int d = 0; d < 8; ++d) {
      int64_t xx = x + moore_dx(d), yy = y + moore_dy(d);
      if (xx >= 0 && yy >= 0 && xx < (int64_t)n && yy < (int64_t)n) c += cur[(uint64_t)yy * n + xx] == 1u;
    }
    next[i] = (uint8_t)rule_byte(v, c, birth, survive);
  }
}

__global__ void k_bb_to_compact(LevelMaps gm, PadLayout L, const uint8_t* __restrict__ grid, uint8_t* __restrict__ st,
                                uint64_t bytes) {
  extern __shared__ uint32_t s_lut[];
  LevelMaps m = stage_maps(gm, s_lut);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < bytes; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t tl = fdiv(L.divKp, i);
    const uint64_t j = i - tl * L.Kp;
    uint8_t v = 0;
    if (j < L.K) {
      uint32_t x, y;
      lambda_level(m, (L.tile_lo + tl) * L.K + j, x, y);
      v = grid[(uint64_t)y * m.n + x];
    }
    st[i] = v;
  }
}

// ---------------------------------------------------------------------------------------
// launchers

static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

static unsigned grid_for(uint64_t work, int threads, int per_sm = 8) {
  uint64_t blocks = (work + threads - 1) / threads;
  uint64_t cap = (uint64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return (unsigned)blocks;
}

static cudaError_t maps_attr(const void* fn, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

cudaError_t launch_map_lambda(const LevelMaps& m, const uint64_t* om, uint32_t* x, uint32_t* y, uint64_t count,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_map_lambda, sm);
  if (e != cudaSuccess) return e;
  k_map_lambda<<<grid_for(count, 256), 256, sm, st>>>(m, om, x, y, count);
  return cudaGetLastError();
}

cudaError_t launch_map_nu(const LevelMaps& m, const uint32_t* x, const uint32_t* y, uint64_t* om, uint64_t count,
                          cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_map_nu, sm);
  if (e != cudaSuccess) return e;
  k_map_nu<<<grid_for(count, 256), 256, sm, st>>>(m, x, y, om, count);
  return cudaGetLastError();
}

static uint64_t splitmix_final(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

cudaError_t launch_seed(const LevelMaps& m, const PadLayout& L, uint8_t* state, uint64_t seed, uint64_t q,
                        cudaStream_t st) {
  const uint64_t words = L.ntiles * L.Kp / 4;
  if (words == 0) return cudaSuccess;
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_seed, sm);
  if (e != cudaSuccess) return e;
  k_seed<<<grid_for(words, 256), 256, sm, st>>>(m, L, words, reinterpret_cast<uint32_t*>(state), splitmix_final(seed),
                                                 q);
  return cudaGetLastError();
}

cudaError_t launch_step_naive(const LevelMaps& m, const uint8_t* cur, uint8_t* next, uint32_t birth, uint32_t survive,
                              const HaloView& halo, cudaStream_t st) {
  const uint64_t words = halo.L.ntiles * halo.L.Kp / 4;
  if (words == 0) return cudaSuccess;
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_step_naive, sm);
  if (e != cudaSuccess) return e;
  k_step_naive<<<grid_for(words, 256), 256, sm, st>>>(m, cur, reinterpret_cast<uint32_t*>(next), words, birth,
                                                       survive, halo);
  return cudaGetLastError();
}

cudaError_t launch_count_alive(const uint8_t* state, uint64_t bytes, uint64_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  uint64_t n16 = bytes / 16;
  uint32_t ntail = (uint32_t)(bytes - n16 * 16);
  k_count_alive<<<grid_for(n16 ? n16 : 1, 256, 4), 256, 0, st>>>(reinterpret_cast<const uint4*>(state), n16,
                                                                  state + n16 * 16, ntail,
                                                                  reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

cudaError_t launch_halo_peer_push(const uint8_t* cur, const uint64_t* send_offsets, const uint32_t* send_peer,
                                  const uint64_t* send_pos, uint64_t nsends, uint8_t* const* peer_recv, cudaStream_t st) {
  if (nsends == 0) return cudaSuccess;
  k_halo_peer_push<<<grid_for(nsends, 256), 256, 0, st>>>(cur, send_offsets, send_peer, send_pos, nsends, peer_recv);
  return cudaGetLastError();
}

cudaError_t launch_halo_pack(const uint8_t* cur, const uint64_t* send_offsets, uint64_t nsends, uint8_t* out,
                             cudaStream_t st) {
  if (nsends == 0) return cudaSuccess;
  k_halo_pack<<<grid_for(nsends, 256), 256, 0, st>>>(cur, send_offsets, nsends, out);
  return cudaGetLastError();
}

cudaError_t launch_bb_seed(const LevelMaps& m, uint8_t* grid, uint64_t seed, uint64_t q, cudaStream_t st) {
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_bb_seed, sm);
  if (e != cudaSuccess) return e;
  k_bb_seed<<<grid_for(m.n * m.n, 256), 256, sm, st>>>(m, grid, m.n, splitmix_final(seed), q);
  return cudaGetLastError();
}

cudaError_t launch_bb_step(const uint8_t* cur, uint8_t* next, uint64_t n, uint32_t birth, uint32_t survive,
                           cudaStream_t st) {
  if (bb_bits_ok(n)) return launch_bb_step_bits(cur, next, n, birth, survive, st);
  k_bb_step1<<<grid_for(n * n, 256), 256, 0, st>>>(cur, next, n, birth, survive);
  return cudaGetLastError();
}

cudaError_t launch_bb_to_compact(const LevelMaps& m, const PadLayout& L, const uint8_t* grid, uint8_t* state,
                                 cudaStream_t st) {
  const uint64_t bytes = L.ntiles * L.Kp;
  if (bytes == 0) return cudaSuccess;
  size_t sm = maps_smem_bytes(m);
  cudaError_t e = maps_attr((const void*)k_bb_to_compact, sm);
  if (e != cudaSuccess) return e;
  k_bb_to_compact<<<grid_for(bytes, 256), 256, sm, st>>>(m, L, grid, state, bytes);
  return cudaGetLastError();
}

}  // namespace sqz
