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
// Stage s swaps the off-diagonal s x s blocks: each lane sends the block its partner keeps
// (a rotate of x & sel) and keeps x & ~sel; 4 instructions per stage.
struct Transposer {
  uint32_t sel[5], amt[5];
  __device__ __forceinline__ explicit Transposer(int lane) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int s = 16 >> k;
      const uint32_t m = (s == 16) ? 0x0000FFFFu : (s == 8) ? 0x00FF00FFu : (s == 4) ? 0x0F0F0F0Fu
                         : (s == 2) ? 0x33333333u : 0x55555555u;
      const bool hi = lane & s;
      sel[k] = hi ? m : ~m;
      amt[k] = hi ? (uint32_t)s : (uint32_t)(32 - s);
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t v = x & sel[k];
      const uint32_t send = __funnelshift_l(v, v, amt[k]);
      x = (x & ~sel[k]) | __shfl_xor_sync(0xFFFFFFFFu, send, 16 >> k);
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

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }
// chunk bytes + slack for the 36-byte windows read past the last tile
__host__ __device__ inline size_t chunk_buf_bytes(uint64_t K) { return align16((size_t)K * kChunkTiles) + 64; }

// Boundary links whose neighbour tile is outside the chunk are prefetched one chunk ahead
// with 4-byte cp.async gathers into R; at most kMaxPrefetchLinks (larger E falls back to a
// synchronous gather).
constexpr uint32_t kMaxPrefetchLinks = 32;

struct TileSmem {
  uint8_t* st0;    // 2 stages x [chunk bytes (input, then output in place) | Z words]
  uint32_t stride, zoff;
  uint16_t* nbr;   // K x 8 neighbour slots into Z
  int64_t* ntl0;   // 2 x [ndirs][32] neighbour tile of each lane's tile (-1 = none)  (producer)
  uint32_t ntn;
  uint32_t* R0;    // 2 x [E][32] prefetched words holding out-of-chunk neighbour bytes (producer)
  uint32_t rn;
  uint64_t* bar;   // [0,2) full (TMA landed), [2,4) links ready, [4,6) output written
  __device__ __forceinline__ uint8_t* buf(int b) const { return st0 + (size_t)b * stride; }
  __device__ __forceinline__ uint32_t* Z(int b) const { return reinterpret_cast<uint32_t*>(st0 + (size_t)b * stride + zoff); }
  __device__ __forceinline__ int64_t* ntl(int b) const { return ntl0 + (size_t)b * ntn; }
  __device__ __forceinline__ uint32_t* R(int b) const { return R0 + (size_t)b * rn; }
};

__host__ __device__ inline uint32_t prefetch_links(const TileParams& p) {
  return p.E <= kMaxPrefetchLinks ? p.E : 0;
}

__host__ __device__ inline size_t tile_layout(const TileParams& p, uint8_t* base, TileSmem* s) {
  const size_t cb = chunk_buf_bytes(p.K), zb = align16((size_t)(p.K + p.E + 1) * 4);
  size_t off = 0;
  if (s) {
    s->st0 = base;
    s->stride = (uint32_t)(cb + zb);
    s->zoff = (uint32_t)cb;
  }
  off += 2 * (cb + zb);
  if (s) s->nbr = (uint16_t*)(base + off);
  off += align16((size_t)p.K * 16);
  const size_t ntn = (size_t)(p.ndirs ? p.ndirs : 1) * kChunkTiles;
  if (s) {
    s->ntl0 = (int64_t*)(base + off);
    s->ntn = (uint32_t)ntn;
  }
  off += 2 * ntn * 8;
  const size_t rn = (size_t)(prefetch_links(p) ? prefetch_links(p) : 1) * kChunkTiles;
  if (s) {
    s->R0 = (uint32_t*)(base + off);
    s->rn = (uint32_t)rn;
  }
  off += 2 * rn * 4;
  if (s) s->bar = (uint64_t*)(base + off);
  off += 6 * 8;
  return align16(off);
}

size_t tile_smem_bytes(const TileParams& p) { return tile_layout(p, nullptr, nullptr); }

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

struct ChunkInfo {
  uint64_t chunk, t0;
  uint32_t nt;
};

__device__ __forceinline__ ChunkInfo chunk_info(const TileParams& p, uint64_t i) {
  ChunkInfo c;
  c.chunk = blockIdx.x + i * gridDim.x;
  c.t0 = p.tile_lo + c.chunk * kChunkTiles;
  c.nt = (uint32_t)min((uint64_t)kChunkTiles, p.tile_hi - c.t0);
  return c;
}

// Producer, lane = tile: coarse λ of the tile (P:212-230 at tile level), then per direction
// the neighbour tile (coarse ν) and, for each link of that direction whose
// neighbour tile lies outside the chunk, an asynchronous 4-byte gather of the word holding
// the neighbour cell's byte (consumed by the same lane in finish_links).
__device__ __forceinline__ void prep_links(const TileParams& p, const TileSmem& S, const ChunkInfo& c, int b,
                                           const uint8_t* __restrict__ cur, int lane) {
  const uint64_t t = c.t0 + lane;
  const uint64_t t_end = c.t0 + c.nt;
  uint32_t X = 0, Y = 0;
  if (t < p.tile_hi) lambda_level(p.coarse, t, X, Y);
  const uint32_t Epf = prefetch_links(p);
  for (uint32_t d = 0; d < p.ndirs; ++d) {
    int64_t tn = -1;
    if (t < p.tile_hi) {
      const uint32_t code = (p.dir_code >> (4 * d)) & 0xFu;
      const int dx = (int)(code & 3u) - 1, dy = (int)(code >> 2) - 1;
      const uint64_t nt = nu_level(p.coarse, (int64_t)X + dx, (int64_t)Y + dy);
      tn = nt == kNoneU64 ? -1 : (int64_t)nt;
    }
    S.ntl(b)[d * kChunkTiles + lane] = tn;
    if (tn >= 0 && ((uint64_t)tn < c.t0 || (uint64_t)tn >= t_end)) {
      const uint32_t e1 = min((uint32_t)p.dir_start[d + 1], Epf);
      for (uint32_t e = p.dir_start[d]; e < e1; ++e) {
        uint32_t* dst = &S.R(b)[e * kChunkTiles + lane];
        const uint64_t om = (uint64_t)tn * p.K + p.link_j2[e];
        if (om >= p.halo.omega_lo && om < p.halo.omega_hi) cp_async4(dst, cur + ((om - p.halo.omega_lo) & ~3ull));
        else *dst = fetch_cell(cur, om, p.halo) << (8 * (uint32_t)(om & 3));  // halo: rare, synchronous
      }
    }
  }
  cp_async_commit();
}

// Producer: one bit-sliced word per tile-boundary link (Z[K+e]) once the chunk has landed.
__device__ __forceinline__ void finish_links(const TileParams& p, const TileSmem& S, const ChunkInfo& c, int b,
                                             const uint8_t* __restrict__ cur, int lane) {
  const uint32_t K = (uint32_t)p.K;
  const uint32_t Epf = prefetch_links(p);
  const uint8_t* buf = S.buf(b);
  uint32_t* Z = S.Z(b);
  cp_async_wait_all();
  for (uint32_t d = 0; d < p.ndirs; ++d) {
    const int64_t tn = S.ntl(b)[d * kChunkTiles + lane];
    const uint64_t rel = (uint64_t)(tn - (int64_t)c.t0);
    const bool inside = tn >= 0 && rel < c.nt;
    const uint32_t lowbase = (uint32_t)tn * K;
    const uint32_t e1 = p.dir_start[d + 1];
    for (uint32_t e = p.dir_start[d]; e < e1; ++e) {
      const uint32_t j2 = p.link_j2[e];
      uint32_t v = 0;
      if (inside) v = buf[(uint32_t)rel * K + j2];
      else if (tn >= 0) {
        if (e < Epf) v = (S.R(b)[e * kChunkTiles + lane] >> (8 * ((lowbase + j2) & 3u))) & 0xFFu;
        else v = fetch_cell(cur, (uint64_t)tn * p.K + j2, p.halo);
      }
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
      if (lane == 0) Z[K + e] = bal;
    }
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&S.bar[2 + b]);
}

// Producer warp: TMA ring (load chunk i+2 as soon as chunk i's output has been read out),
// link prefetch two chunks ahead, link words one chunk ahead.
__device__ __forceinline__ void producer(const TileParams& p, const TileSmem& S, const uint8_t* __restrict__ cur,
                                         uint8_t* __restrict__ next, int lane, uint64_t n) {
  const uint32_t K = (uint32_t)p.K;
  auto load = [&](uint64_t i) {
    const ChunkInfo c = chunk_info(p, i);
    const int b = (int)(i & 1);
    if (lane == 0) {
      fence_proxy_async();
      tma_load_1d(S.buf(b), cur + c.chunk * kChunkTiles * p.K, (uint32_t)align16((size_t)c.nt * K), &S.bar[b]);
    }
    prep_links(p, S, c, b, cur, lane);
  };
  load(0);
  if (n > 1) load(1);
  mbar_wait(&S.bar[0], 0);
  finish_links(p, S, chunk_info(p, 0), 0, cur, lane);
  for (uint64_t i = 0; i < n; ++i) {
    const int b = (int)(i & 1);
    const uint32_t u = (uint32_t)((i >> 1) & 1);
    if (i + 1 < n) {  // link words of the next chunk (its data landed a chunk ago)
      mbar_wait(&S.bar[b ^ 1], (uint32_t)(((i + 1) >> 1) & 1));
      finish_links(p, S, chunk_info(p, i + 1), b ^ 1, cur, lane);
    }
    mbar_wait(&S.bar[4 + b], u);  // consumers wrote chunk i's output
    const ChunkInfo c = chunk_info(p, i);
    if (lane == 0) {
      tma_store_1d(next + c.chunk * kChunkTiles * p.K, S.buf(b), (uint32_t)align16((size_t)c.nt * K));
      if (i + 2 < n) bulk_wait_read_all();
    }
    __syncwarp();
    if (i + 2 < n) load(i + 2);
  }
  cp_async_wait_all();
  if (lane == 0) bulk_wait_all();
}

// MAXT/MINB: launch bounds; the default 288-thread shape is compiled for 3 CTAs per SM.
template <int DMAX, bool CONWAY, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_step_tile(TileParams p, const uint8_t* __restrict__ cur,
                                                         uint8_t* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TileSmem S;
  tile_layout(p, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NC = (int)(blockDim.x >> 5) - 1;  // consumer warps; the last warp produces
  const uint32_t K = (uint32_t)p.K;
  const uint32_t nblk = (K + 31) / 32;
  const uint64_t n = p.nchunks > blockIdx.x ? (p.nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  {
    const uint4* src = reinterpret_cast<const uint4*>(p.nbr);
    uint4* dst = reinterpret_cast<uint4*>(S.nbr);
    for (uint32_t i = tid; i < K; i += blockDim.x) dst[i] = src[i];
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.bar[b], 1);
      mbar_init(&S.bar[2 + b], 1);
      mbar_init(&S.bar[4 + b], (uint32_t)NC);
      S.Z(b)[p.zslot] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (n == 0) return;
  if (warp == NC) {
    producer(p, S, cur, next, lane, n);
    return;
  }

  // ---------------------------------------------------------------- consumer warps
  uint32_t tail_mask = 0;  // packed bits (bit 8p+m = cell 4m+p) valid in the last j-block
  {
    const uint32_t nv = K - (nblk - 1) * 32;
#pragma unroll
    for (int b = 0; b < 32; ++b)
      if ((uint32_t)(4 * (b & 7) + (b >> 3)) < nv) tail_mask |= 1u << b;
  }
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);  // cell offset this lane holds after a transpose
  const Transposer tr(lane);
  const int nct = NC * 32;

  for (uint64_t i = 0; i < n; ++i) {
    const int b = (int)(i & 1);
    const uint32_t u = (uint32_t)((i >> 1) & 1);
    const ChunkInfo c = chunk_info(p, i);
    const bool active = (uint32_t)lane < c.nt;
    uint8_t* inb = S.buf(b);
    uint32_t* Z = S.Z(b);
    const uint32_t* in32 = reinterpret_cast<const uint32_t*>(inb);
    mbar_wait(&S.bar[b], u);

    // Phase A: lane = tile; 32 bytes (cells j0..j0+31) -> bits 8p+m = cell 4m+p -> transpose,
    // leaving lane L with the bit-sliced word of cell j0 + my_jj(L)
    for (uint32_t jb = warp; jb < nblk; jb += NC) {
      const uint32_t j0 = jb * 32;
      const uint32_t a = (uint32_t)lane * K + j0;
      const uint32_t wi = a >> 2, sh = (a & 3) * 8;
      uint32_t w[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) w[m] = in32[wi + m];
      uint32_t acc = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m) acc += (__funnelshift_r(w[m], w[m + 1], sh) & 0x01010101u) << m;
      if (jb == nblk - 1) acc &= tail_mask;
      if (!active) acc = 0;
      const uint32_t x = tr(acc);
      if (j0 + my_jj < K) Z[j0 + my_jj] = x;
    }
    consumer_sync(nct);             // all state words of the chunk are in Z
    mbar_wait(&S.bar[2 + b], u);    // the producer wrote the link words

    // Phases C + D per j-block: lane L computes cell j0 + my_jj(L) of all 32 tiles (carry-save
    // count, rule), then the block is transposed back (lane = tile) and written in place
    const uint32_t live_lanes = c.nt >= 32 ? 0xFFFFFFFFu : ((1u << c.nt) - 1u);
    for (uint32_t jb = warp; jb < nblk; jb += NC) {
      const uint32_t j0 = jb * 32;
      const uint32_t j = j0 + my_jj;
      uint32_t nw = 0;
      if (j < K) {
        const uint4 row = reinterpret_cast<const uint4*>(S.nbr)[j];
        uint32_t x[8];
        x[0] = Z[row.x & 0xFFFFu];
        x[1] = Z[row.x >> 16];
        x[2] = Z[row.y & 0xFFFFu];
        x[3] = Z[row.y >> 16];
        x[4] = Z[row.z & 0xFFFFu];
        if (DMAX > 5) {
          x[5] = Z[row.z >> 16];
          x[6] = Z[row.w & 0xFFFFu];
          x[7] = Z[row.w >> 16];
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
        const uint32_t alive = Z[j];
        if (CONWAY) {
          nw = c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23: count 3, or count 2 and alive
        } else {
          nw = (alive & rule_bits(p.survive, c0, c1, c2, c3)) | (~alive & rule_bits(p.birth, c0, c1, c2, c3));
        }
        nw &= live_lanes;
      }
      const uint32_t xb = tr(nw);  // bit 8p+m = cell j0 + 4m + p of this lane's tile
      if (!active) continue;
      const uint32_t a = (uint32_t)lane * K + j0;
      const uint32_t nv = min(32u, K - j0);
      uint32_t bw[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) bw[m] = (xb >> m) & 0x01010101u;
      if (nv == 32) {
        const uint32_t sh = a & 3;
        uint32_t* out32 = reinterpret_cast<uint32_t*>(inb + (a - sh));
        if (sh == 0) {
#pragma unroll
          for (int m = 0; m < 8; ++m) out32[m] = bw[m];
        } else {
          const uint32_t d = 4 - sh;  // bytes before the first aligned word (byte stores)
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if ((uint32_t)q < d) inb[a + q] = (uint8_t)(bw[0] >> (8 * q));
#pragma unroll
          for (int k = 1; k < 8; ++k) out32[k] = __funnelshift_r(bw[k - 1], bw[k], 8 * d);
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
    if (warp == 0) {  // zero padding up to the 16-byte bulk-copy granule
      const uint32_t bytes = c.nt * K;
      const uint32_t padded = (uint32_t)align16(bytes);
      if (bytes + lane < padded) inb[bytes + lane] = 0;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.bar[4 + b]);
  }
}

// ---------------------------------------------------------------------------------------

using TileFn = void (*)(TileParams, const uint8_t*, uint8_t*);

static TileFn pick(const TileParams& p, int threads) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  if (threads <= 288) {
    if (p.dmax <= 5) return conway ? k_step_tile<5, true, 288, 3> : k_step_tile<5, false, 288, 3>;
    return conway ? k_step_tile<8, true, 288, 3> : k_step_tile<8, false, 288, 3>;
  }
  if (p.dmax <= 5) return conway ? k_step_tile<5, true, 1024, 1> : k_step_tile<5, false, 1024, 1>;
  return conway ? k_step_tile<8, true, 1024, 1> : k_step_tile<8, false, 1024, 1>;
}

cudaError_t tile_prepare(const TileParams& p, size_t smem, int threads, int* occupancy) {
  TileFn fn = pick(p, threads);
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
  pick(p, threads)<<<grid, threads, smem, st>>>(p, cur, next);
  return cudaGetLastError();
}

}  // namespace sqz
