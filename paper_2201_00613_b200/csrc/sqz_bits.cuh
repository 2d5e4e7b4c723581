// sqz_bits.cuh — device building blocks shared by the byte-state and packed-state tile kernels
// (internal): TMA/mbarrier/cp.async wrappers, the warp bit transpose, bit-sliced counting and
// rule evaluation, chunk bookkeeping and the coarse maps of a chunk's 32 tiles.
#pragma once

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
// Stage s exchanges the off-diagonal s x s bit blocks between lanes L and L^s: the lane with
// (L & s) == 0 keeps its bits {b : (b & s) == 0} and takes the partner's same bits moved up by
// s; the other lane keeps {b : b & s} and takes the partner's moved down by s.  Every lane
// sends its raw word.  s = 16, 8 move whole bytes: one PRMT picks the kept and received bytes.
// s = 4, 2, 1: rotate the received word by +-s (per-lane amount) and merge with one LOP3.
struct Transposer {
  uint32_t perm16, perm8;  // PRMT selectors
  uint32_t keep[3], amt[3];
  __device__ __forceinline__ explicit Transposer(int lane) {
    perm16 = (lane & 16) ? 0x3276u : 0x5410u;  // hi: [r2 r3 x2 x3]   lo: [x0 x1 r0 r1]
    perm8 = (lane & 8) ? 0x3715u : 0x6240u;    // hi: [r1 x1 r3 x3]   lo: [x0 r0 x2 r2]
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = 4 >> k;
      const uint32_t m = (s == 4) ? 0x0F0F0F0Fu : (s == 2) ? 0x33333333u : 0x55555555u;
      const bool hi = lane & s;
      keep[k] = hi ? ~m : m;
      amt[k] = hi ? (uint32_t)(32 - s) : (uint32_t)s;
    }
    // Identity shuffles make the constants opaque, so ptxas keeps them in registers instead
    // of re-deriving them from the lane id inside the hot loops.
    perm16 = __shfl_sync(0xFFFFFFFFu, perm16, lane);
    perm8 = __shfl_sync(0xFFFFFFFFu, perm8, lane);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      keep[k] = __shfl_sync(0xFFFFFFFFu, keep[k], lane);
      amt[k] = __shfl_sync(0xFFFFFFFFu, amt[k], lane);
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    x = __byte_perm(x, __shfl_xor_sync(0xFFFFFFFFu, x, 16), perm16);
    x = __byte_perm(x, __shfl_xor_sync(0xFFFFFFFFu, x, 8), perm8);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t r = __shfl_xor_sync(0xFFFFFFFFu, x, 4 >> k);
      const uint32_t rot = __funnelshift_l(r, r, amt[k]);
      x = (x & keep[k]) | (rot & ~keep[k]);
    }
    return x;
  }
};

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

// Shared-memory accesses by 32-bit shared-window address (no generic->shared conversion per use).
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// 32 state bytes (cells c..c+31 of one tile, each 0 or 1 by the input contract) -> 32 bits,
// bit 8p+m = cell 4m+p.  Shifted adds (LEA) never carry between bytes for 0/1 inputs.
__device__ __forceinline__ uint32_t pack01(const uint4& lo, const uint4& hi) {
  uint32_t a = lo.x + (lo.y << 1);
  a += lo.z << 2;
  a += lo.w << 3;
  a += hi.x << 4;
  a += hi.y << 5;
  a += hi.z << 6;
  a += hi.w << 7;
  return a;
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// Boundary links whose neighbour tile is outside the chunk are prefetched one chunk ahead
// with 4-byte cp.async gathers into R; at most kMaxPrefetchLinks (larger E falls back to a
// synchronous gather).
constexpr uint32_t kMaxPrefetchLinks = 160;

__host__ __device__ inline uint32_t prefetch_links(const TileParams& p) {
  return p.E <= kMaxPrefetchLinks ? p.E : 0;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// 4-byte cp.async issued only where `pred` is set (a predicated instruction, no branch)
__device__ __forceinline__ void cp_async4_if(uint32_t dst, const void* src, uint32_t pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.ca.shared.global [%0], [%1], 4;\n\t}" ::"r"(dst),
      "l"(src), "r"(pred)
      : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct ChunkInfo {
  uint64_t chunk, t0;
  uint32_t nt;
};

__device__ __forceinline__ ChunkInfo chunk_info(const TileParams& p, uint64_t chunk) {
  ChunkInfo c;
  c.chunk = chunk;
  c.t0 = p.tile_lo + chunk * kChunkTiles;
  c.nt = (uint32_t)min((uint64_t)kChunkTiles, p.tile_hi - c.t0);
  return c;
}

// Dynamic j-block distribution: warps that carry extra work (coarse maps, TMA) take fewer blocks.
__device__ __forceinline__ uint32_t grab(uint32_t ctr_s, int lane) {  // ctr_s: shared-window address
  uint32_t v = 0;
  if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(v) : "r"(ctr_s) : "memory");
  return __shfl_sync(0xFFFFFFFFu, v, 0);
}
__device__ __forceinline__ uint32_t grab(uint32_t* ctr, int lane) { return grab(smem_u32(ctr), lane); }

// Warp w, directions d = w, w + nwarps, ...: neighbour tile of each lane's tile (from the
// adjacency table: coarse λ then coarse ν, P:189 at tile level, evaluated once at init) and,
// for each link of direction d whose neighbour tile is outside the chunk, a 4-byte cp.async
// gather of the word holding the neighbour cell.  The same warp consumes them in Phase B of
// that chunk.  Always commits exactly one group.
// Tile-padded byte layout: the gather fetches the aligned word holding the byte.
__device__ __forceinline__ void chunk_neighbours(const TileParams& p, uint32_t* ntl, uint32_t* R, const uint32_t* lj2,
                                                 const ChunkInfo& c, const uint8_t* __restrict__ cur, int warp,
                                                 int nwarps, int lane, uint32_t Epf) {
  const uint64_t t = c.t0 + lane;
  const uint64_t t_end = c.t0 + c.nt;
  for (int d = warp; d < (int)p.ndirs; d += nwarps) {
    const uint32_t a1 = (t < p.tile_hi) ? __ldg(p.adj + d * p.adj_stride + (t - p.tile_lo)) : 0u;
    const int64_t tn = (int64_t)a1 - 1;
    ntl[d * kChunkTiles + lane] = a1;  // tiles < 2^32 - 1 (checked on the host)
    if (tn >= 0 && ((uint64_t)tn < c.t0 || (uint64_t)tn >= t_end)) {
      const uint32_t e1 = min(lj2[p.E + d + 1], Epf);  // lj2: [E] link cells, then direction starts
      for (uint32_t e = lj2[p.E + d]; e < e1; ++e) {
        uint32_t* dst = &R[e * kChunkTiles + lane];
        const uint32_t j2 = lj2[e];
        if ((uint64_t)tn >= p.tile_lo && (uint64_t)tn < p.tile_hi) {
          const uint64_t off = ((uint64_t)tn - p.tile_lo) * p.Kp + j2;
          cp_async4(dst, cur + (off & ~3ull));
        } else {
          *dst = fetch_cell(cur, (uint64_t)tn * p.K + j2, p.halo) << (8 * (j2 & 3u));  // halo: rare, synchronous
        }
      }
    }
  }
  cp_async_commit();
}

__device__ __forceinline__ void chunk_neighbours(const TileParams& p, uint32_t* ntl, uint32_t* R, const uint32_t* lj2,
                                                 const ChunkInfo& c, const uint8_t* __restrict__ cur, int warp,
                                                 int nwarps, int lane) {
  chunk_neighbours(p, ntl, R, lj2, c, cur, warp, nwarps, lane, prefetch_links(p));
}

}  // namespace sqz
