// sqz_tile.cu — the product stencil kernel: one automaton step on the compact array,
// tile-amortised and bit-sliced.
//
// Work unit ("chunk"): 32 consecutive level-g tiles = 32·K contiguous bytes of Ω order.
// Every level-g tile is a translated copy of the same sub-fractal (NBB class), so
// the neighbour of local cell j is the same local cell j' in every tile (one shared table)
// except for the few tile-boundary links, whose neighbour tile comes from one coarse λ and
// one coarse ν per tile (P:189 applied at block level).  Bit i of a 32-bit word is
// tile i of the chunk, so one word op updates 32 cells.
//
//   TMA 1D bulk copy  global -> smem          (cp.async.bulk + mbarrier, 1 chunk ahead)
//   Phase A  bytes -> bit-sliced words Z[j]   (funnel shift, OR-pack, 32x32 shuffle transpose)
//   Phase B  boundary-link words Z[K+e]       (ballot of the neighbour tile's cell, per lane)
//   Phase C  count (carry-save adders) + rule W[j]
//   Phase D  W -> bytes in place              (shuffle transpose, unpack, aligned stores)
//   TMA 1D bulk copy  smem -> global
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_device.cuh"
#include "sqz_kernels.cuh"

namespace sqz {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32x32 bit transpose across the warp: afterwards lane L bit i = (lane i bit L) before.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = (s == 16) ? 0x0000FFFFu : (s == 8) ? 0x00FF00FFu : (s == 4) ? 0x0F0F0F0Fu
                       : (s == 2) ? 0x33333333u : 0x55555555u;
    uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
  }
  return x;
}

// Bit-sliced rule f(c) = bit c of `mask` (c <= 8), a mux tree on the count bits.
__device__ __forceinline__ uint32_t mask_word(uint32_t mask, int v) { return ((mask >> v) & 1u) ? 0xFFFFFFFFu : 0u; }

__device__ __forceinline__ uint32_t rule_bits(uint32_t mask, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  uint32_t m0 = (mask_word(mask, 0) & ~c0) | (mask_word(mask, 1) & c0);
  uint32_t m1 = (mask_word(mask, 2) & ~c0) | (mask_word(mask, 3) & c0);
  uint32_t m2 = (mask_word(mask, 4) & ~c0) | (mask_word(mask, 5) & c0);
  uint32_t m3 = (mask_word(mask, 6) & ~c0) | (mask_word(mask, 7) & c0);
  uint32_t m4 = mask_word(mask, 8) & ~c0;
  uint32_t n0 = (m0 & ~c1) | (m1 & c1);
  uint32_t n1 = (m2 & ~c1) | (m3 & c1);
  uint32_t n2 = m4 & ~c1;
  uint32_t o0 = (n0 & ~c2) | (n1 & c2);
  uint32_t o1 = n2 & ~c2;
  return (o0 & ~c3) | (o1 & c3);
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

struct TileSmem {
  uint8_t* in0;       // 2 chunk buffers of `cb` bytes (each reused in place for the output)
  uint32_t cb;
  uint32_t* Z;        // K state words | E link words | zero word
  uint32_t* W;        // K next words
  uint16_t* nbr;      // K x 8 neighbour slots into Z
  int64_t* nt0;       // 2 x [ndirs][32] neighbour tile of each lane's tile, -1 = none
  uint32_t ntn;       // int64 entries per ntile buffer
  uint64_t* bar;      // 2 mbarriers
  __device__ __forceinline__ uint8_t* in(int b) const { return in0 + (size_t)b * cb; }
  __device__ __forceinline__ int64_t* ntile(int b) const { return nt0 + (size_t)b * ntn; }
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }
// chunk bytes + slack for the 36-byte windows of the last tile
__host__ __device__ inline size_t chunk_buf_bytes(uint64_t K) { return align16((size_t)K * kChunkTiles) + 64; }

__host__ __device__ inline size_t tile_layout(const TileParams& p, uint8_t* base, TileSmem* s) {
  size_t off = 0;
  size_t cb = chunk_buf_bytes(p.K);
  if (s) {
    s->in0 = base + off;
    s->cb = (uint32_t)cb;
  }
  off += 2 * cb;
  if (s) s->Z = (uint32_t*)(base + off);
  off += align16((size_t)(p.K + p.E + 1) * 4);
  if (s) s->W = (uint32_t*)(base + off);
  off += align16((size_t)p.K * 4);
  if (s) s->nbr = (uint16_t*)(base + off);
  off += align16((size_t)p.K * 16);
  size_t nt = (size_t)(p.ndirs ? p.ndirs : 1) * kChunkTiles * 8;
  if (s) {
    s->nt0 = (int64_t*)(base + off);
    s->ntn = (uint32_t)(nt / 8);
  }
  off += 2 * nt;
  if (s) s->bar = (uint64_t*)(base + off);
  off += 16;
  return off;
}

size_t tile_smem_bytes(const TileParams& p) { return tile_layout(p, nullptr, nullptr); }

// Warp w < ndirs: for each lane's tile of chunk `chunk`, the neighbour tile in direction w
// (coarse λ then coarse ν, P:189 at tile granularity), or -1.
__device__ __forceinline__ void compute_ntile_dir(const TileParams& p, uint64_t chunk, int64_t* dst, int dir,
                                                  int lane) {
  uint64_t t = p.tile_lo + chunk * kChunkTiles + lane;
  int64_t v = -1;
  if (t < p.tile_hi) {
    uint32_t X, Y;
    lambda_level(p.coarse, t, X, Y);
    const uint32_t code = (p.dir_code >> (4 * dir)) & 0xFu;
    const int dx = (int)(code & 3u) - 1, dy = (int)(code >> 2) - 1;
    uint64_t nt = nu_level(p.coarse, (int64_t)X + dx, (int64_t)Y + dy);
    v = (nt == kNoneU64) ? -1 : (int64_t)nt;
  }
  dst[dir * kChunkTiles + lane] = v;
}

template <int DMAX, bool CONWAY>
__global__ void __launch_bounds__(1024) k_step_tile(TileParams p, const uint8_t* __restrict__ cur,
                                                    uint8_t* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TileSmem S;
  tile_layout(p, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K;
  const uint32_t nblk = (K + 31) / 32;
  // bits of the packed layout (bit 8p+m = cell 4m+p) that are valid in the last j-block
  uint32_t tail_mask = 0;
  {
    const uint32_t nv = K - (nblk - 1) * 32;
#pragma unroll
    for (int b = 0; b < 32; ++b)
      if ((uint32_t)(4 * (b & 7) + (b >> 3)) < nv) tail_mask |= 1u << b;
  }
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);  // cell offset this lane owns after a transpose

  {
    const uint4* src = reinterpret_cast<const uint4*>(p.nbr);
    uint4* dst = reinterpret_cast<uint4*>(S.nbr);
    for (uint32_t i = tid; i < K; i += blockDim.x) dst[i] = src[i];
  }
  if (tid == 0) {
    S.Z[p.zslot] = 0;
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t chunk = blockIdx.x;
  if (chunk < p.nchunks) {
    if (tid == 0) {
      uint64_t t0 = p.tile_lo + chunk * kChunkTiles;
      uint64_t nt = min((uint64_t)kChunkTiles, p.tile_hi - t0);
      tma_load_1d(S.in(0), cur + chunk * kChunkTiles * p.K, (uint32_t)align16(nt * p.K), &S.bar[0]);
    }
    if (warp < (int)p.ndirs) compute_ntile_dir(p, chunk, S.ntile(0), warp, lane);
  }
  __syncthreads();

  uint32_t it = 0;
  for (; chunk < p.nchunks; chunk += gridDim.x, ++it) {
    const int buf = it & 1;
    const uint64_t t0 = p.tile_lo + chunk * kChunkTiles;
    const uint32_t nt = (uint32_t)min((uint64_t)kChunkTiles, p.tile_hi - t0);
    const uint64_t nxt = chunk + gridDim.x;
    if (nxt < p.nchunks) {
      if (tid == 0) {
        // in[buf^1] held the previous chunk's output: its bulk store must have read it
        bulk_wait_read_all();
        uint64_t n0 = p.tile_lo + nxt * kChunkTiles;
        uint64_t nn = min((uint64_t)kChunkTiles, p.tile_hi - n0);
        fence_proxy_async();
        tma_load_1d(S.in(buf ^ 1), cur + nxt * kChunkTiles * p.K, (uint32_t)align16(nn * p.K), &S.bar[buf ^ 1]);
      }
      if (warp < (int)p.ndirs) compute_ntile_dir(p, nxt, S.ntile(buf ^ 1), warp, lane);
    }
    mbar_wait(&S.bar[buf], (it >> 1) & 1);
    uint8_t* inb = S.in(buf);
    const uint32_t* in32 = reinterpret_cast<const uint32_t*>(inb);
    const bool active = (uint32_t)lane < nt;

    // Phase A: lane = tile.  32 bytes (cells j0..j0+31) -> 32 bits, bit 8p+m = cell 4m+p,
    // then a 32x32 transpose leaves lane L with the word of cell j0 + my_jj(L).
    for (uint32_t jb = warp; jb < nblk; jb += nwarps) {
      const uint32_t j0 = jb * 32;
      const uint32_t a = (uint32_t)lane * K + j0;
      const uint32_t wi = a >> 2, sh = (a & 3) * 8;
      uint32_t w[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) w[m] = in32[wi + m];
      uint32_t acc = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m) acc |= (__funnelshift_r(w[m], w[m + 1], sh) & 0x01010101u) << m;
      if (jb == nblk - 1) acc &= tail_mask;
      if (!active) acc = 0;
      uint32_t x = transpose32(acc, lane);
      if (j0 + my_jj < K) S.Z[j0 + my_jj] = x;
    }
    // Phase B: tile-boundary links; lane i reads its neighbour tile's cell j2
    {
      const int64_t* ntl = S.ntile(buf);
      for (uint32_t e = warp; e < p.E; e += nwarps) {
        const uint32_t d = p.link_dir[e], j2 = p.link_j2[e];
        const int64_t tn = ntl[d * kChunkTiles + lane];
        uint32_t v = 0;
        if (tn >= 0) {
          const uint64_t tu = (uint64_t)tn;
          if (tu >= t0 && tu < t0 + nt) v = inb[(size_t)(tu - t0) * K + j2];
          else v = fetch_cell(cur, tu * p.K + j2, p.halo);
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
        if (lane == 0) S.Z[K + e] = bal;
      }
    }
    __syncthreads();

    // Phase C: lane = cell j of all 32 tiles; carry-save count of <= DMAX neighbour words
    const uint32_t live_lanes = nt >= 32 ? 0xFFFFFFFFu : ((1u << nt) - 1u);
    for (uint32_t j = tid; j < K; j += blockDim.x) {
      const uint4 row = reinterpret_cast<const uint4*>(S.nbr)[j];
      uint32_t x[8];
      x[0] = S.Z[row.x & 0xFFFFu];
      x[1] = S.Z[row.x >> 16];
      x[2] = S.Z[row.y & 0xFFFFu];
      x[3] = S.Z[row.y >> 16];
      x[4] = S.Z[row.z & 0xFFFFu];
      if (DMAX > 5) {
        x[5] = S.Z[row.z >> 16];
        x[6] = S.Z[row.w & 0xFFFFu];
        x[7] = S.Z[row.w >> 16];
      }
      uint32_t c0, c1, c2, c3;
      if (DMAX <= 5) {
        const uint32_t s1 = x[0] ^ x[1] ^ x[2], k1 = maj3(x[0], x[1], x[2]);
        const uint32_t s2 = s1 ^ x[3] ^ x[4], k2 = maj3(s1, x[3], x[4]);
        c0 = s2;
        c1 = k1 ^ k2;
        c2 = k1 & k2;
        c3 = 0;
      } else {
        const uint32_t sa = x[0] ^ x[1] ^ x[2], ka = maj3(x[0], x[1], x[2]);
        const uint32_t sb = x[3] ^ x[4] ^ x[5], kb = maj3(x[3], x[4], x[5]);
        const uint32_t sc = sa ^ sb ^ x[6], kc = maj3(sa, sb, x[6]);
        c0 = sc ^ x[7];
        const uint32_t kd = sc & x[7];
        const uint32_t se = ka ^ kb ^ kc, ke = maj3(ka, kb, kc);
        c1 = se ^ kd;
        const uint32_t kf = se & kd;
        c2 = ke ^ kf;
        c3 = ke & kf;
      }
      const uint32_t alive = S.Z[j];
      uint32_t nw;
      if (CONWAY) {
        nw = c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23: count 3, or count 2 and alive
      } else {
        nw = (alive & rule_bits(p.survive, c0, c1, c2, c3)) | (~alive & rule_bits(p.birth, c0, c1, c2, c3));
      }
      S.W[j] = nw & live_lanes;
    }
    __syncthreads();

    // Phase D: transpose back (lane = tile) and write the 32 bytes of each j-block in place
    for (uint32_t jb = warp; jb < nblk; jb += nwarps) {
      const uint32_t j0 = jb * 32;
      uint32_t x = (j0 + my_jj < K) ? S.W[j0 + my_jj] : 0u;
      x = transpose32(x, lane);  // bit 8p+m = cell j0 + 4m + p of this lane's tile
      if (!active) continue;
      const uint32_t a = (uint32_t)lane * K + j0;
      const uint32_t nv = min(32u, K - j0);
      uint32_t bw[9];
#pragma unroll
      for (int m = 0; m < 8; ++m) bw[m] = (x >> m) & 0x01010101u;
      bw[8] = 0;
      if (nv == 32) {
        const uint32_t sh = a & 3;
        uint32_t* out32 = reinterpret_cast<uint32_t*>(inb + (a - sh));
        if (sh == 0) {
#pragma unroll
          for (int m = 0; m < 8; ++m) out32[m] = bw[m];
        } else {
          const uint32_t d = 4 - sh;  // bytes before the first aligned word
          // head: bytes 0..d-1 go to the tail of word out32[0]
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if ((uint32_t)q < d) inb[a + q] = (uint8_t)(bw[0] >> (8 * q));
          // body: aligned words 1..7 hold bytes d + 4(k-1) .. d + 4(k-1) + 3
#pragma unroll
          for (int k = 1; k < 8; ++k) out32[k] = __funnelshift_r(bw[k - 1], bw[k], 8 * d);
          // tail: the last sh bytes (q = 32 - sh .. 31) live in bw[7] bytes (4 - sh) .. 3
#pragma unroll
          for (int q = 1; q < 4; ++q)
            if ((uint32_t)q >= d) inb[a + 28 + q] = (uint8_t)(bw[7] >> (8 * q));
        }
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if ((uint32_t)q < nv) inb[a + q] = (uint8_t)(bw[q >> 2] >> (8 * (q & 3)));
      }
    }
    const uint32_t bytes = nt * K;
    const uint32_t padded = (uint32_t)align16(bytes);
    for (uint32_t i = bytes + tid; i < padded; i += blockDim.x) inb[i] = 0;
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) tma_store_1d(next + chunk * kChunkTiles * p.K, inb, padded);
  }
  if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------------------

using TileFn = void (*)(TileParams, const uint8_t*, uint8_t*);

static TileFn pick(const TileParams& p) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  if (p.dmax <= 5) return conway ? k_step_tile<5, true> : k_step_tile<5, false>;
  return conway ? k_step_tile<8, true> : k_step_tile<8, false>;
}

cudaError_t tile_prepare(const TileParams& p, size_t smem, int threads, int* occupancy) {
  TileFn fn = pick(p);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t launch_step_tile(const TileParams& p, const uint8_t* cur, uint8_t* next, int grid, int threads,
                             size_t smem, cudaStream_t st) {
  if (p.nchunks == 0) return cudaSuccess;
  pick(p)<<<grid, threads, smem, st>>>(p, cur, next);
  return cudaGetLastError();
}

}  // namespace sqz
