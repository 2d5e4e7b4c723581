// sqz_packed.cu — the automaton step on the BIT-SLICED PACKED state.
//
// Packed layout (include/squeeze.h): chunk c of a shard = its 32 consecutive level-g tiles;
// Kw = round_up(K, 4) 32-bit words per chunk; word j bit i = cell j of tile 32c + i.  This is
// exactly the bit-sliced form the byte-state kernel (sqz_tile.cu) builds in shared memory, so
// here a step is: TMA the chunk's words in, add one word per tile-boundary link, carry-save
// count + rule per word (32 cells), TMA the words out.  1 bit per cell in HBM (0.25 B/cell of
// traffic per step instead of 2 B) and no byte<->bit staging.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_bits.cuh"

namespace sqz {

// ------------------------------------------------------------------------------------ layout
struct PackedSmem {
  uint32_t* Zin0;   // 2 x [Kw state words (TMA target) | E link words | zero word]
  uint32_t zn;
  uint32_t* Zout0;  // 2 x [Kw next-state words] (TMA source)
  uint32_t* ntl;    // [ndirs][32] neighbour tile + 1 (next chunk)
  uint32_t* R;      // [E][32] prefetched words (next chunk)
  uint64_t* bar;    // [0,2) TMA load landed, [2,4) all warps wrote Zout
  uint32_t* ctr;    // [2] block counters by chunk parity
  __device__ __forceinline__ uint32_t* Zin(int b) const { return Zin0 + (size_t)b * zn; }
  __device__ __forceinline__ uint32_t* Zout(int b) const { return Zout0 + (size_t)b * zn; }
};

__host__ __device__ inline size_t packed_layout(const TileParams& p, uint8_t* base, PackedSmem* s) {
  const size_t zn = align16((size_t)(p.Kw + p.E + 1) * 4) / 4;
  size_t off = 0;
  if (s) {
    s->Zin0 = (uint32_t*)base;
    s->zn = (uint32_t)zn;
  }
  off += 2 * zn * 4;
  if (s) s->Zout0 = (uint32_t*)(base + off);
  off += 2 * zn * 4;
  if (s) s->ntl = (uint32_t*)(base + off);
  off += (size_t)(p.ndirs ? p.ndirs : 1) * kChunkTiles * 4;
  if (s) s->R = (uint32_t*)(base + off);
  off += (size_t)(prefetch_links(p) ? prefetch_links(p) : 1) * kChunkTiles * 4;
  if (s) s->bar = (uint64_t*)(base + off);
  off += 32;
  if (s) s->ctr = (uint32_t*)(base + off);
  off += 16;
  return align16(off);
}

size_t packed_smem_bytes(const TileParams& p) { return packed_layout(p, nullptr, nullptr); }

// ------------------------------------------------------------------------------------ step
template <int DMAX, bool CONWAY>
__global__ void __launch_bounds__(256, 4) k_step_packed(TileParams p, const uint32_t* __restrict__ cur,
                                                        uint32_t* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PackedSmem S;
  packed_layout(p, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K, Kw = p.Kw;
  const uint32_t nblk = (K + 31) / 32;
  const uint32_t Epf = prefetch_links(p);
  const int lw = nwarps - 1;
  const bool issuer = warp == lw && lane == 0;
  const uint8_t* cur8 = reinterpret_cast<const uint8_t*>(cur);

  for (uint32_t i = tid; i < 2 * S.zn; i += blockDim.x) S.Zout0[i] = 0;  // padding words stay 0
  if (tid == 0) {
    S.Zin(0)[Kw + p.E] = 0;
    S.Zin(1)[Kw + p.E] = 0;
    S.ctr[0] = S.ctr[1] = 0;
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init(&S.bar[2], (uint32_t)nwarps);
    mbar_init(&S.bar[3], (uint32_t)nwarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t chunk = blockIdx.x;
  if (chunk >= p.nchunks) return;
  const uint64_t G = gridDim.x;
  const uint32_t cbytes = Kw * 4;
  {  // prologue: chunk 0 loaded, λ of chunks 0 and 1, neighbours + prefetch of chunk 0
    const ChunkInfo c0 = chunk_info(p, chunk);
    if (issuer) tma_load_1d(S.Zin(0), cur + chunk * Kw, cbytes, &S.bar[0]);
    chunk_neighbours<true>(p, S.ntl, S.R, c0, cur8, warp, nwarps, lane);
  }

  uint32_t it = 0;
  for (; chunk < p.nchunks; chunk += G, ++it) {
    const int buf = it & 1;
    const ChunkInfo c = chunk_info(p, chunk);
    const bool has_next = chunk + G < p.nchunks;
    if (issuer) {
      if (it >= 1) {  // the previous chunk is complete: write it out, then reuse its input buffer
        mbar_wait(&S.bar[2 + (buf ^ 1)], ((it - 1) >> 1) & 1);
        tma_store_1d(next + (chunk - G) * Kw, S.Zout(buf ^ 1), cbytes);
      }
      if (has_next) {
        fence_proxy_async();
        tma_load_1d(S.Zin(buf ^ 1), cur + (chunk + G) * Kw, cbytes, &S.bar[buf ^ 1]);
      }
    }
    mbar_wait(&S.bar[buf], (it >> 1) & 1);
    uint32_t* Z = S.Zin(buf);

    // link words: bit i of Z[Kw + e] = cell j2 of lane i's neighbour tile in the link's direction
    if (warp < (int)p.ndirs) {
      cp_async_wait_all();
      for (int d = warp; d < (int)p.ndirs; d += nwarps) {
        const int64_t tn = (int64_t)S.ntl[d * kChunkTiles + lane] - 1;
        const uint64_t rel = (uint64_t)(tn - (int64_t)c.t0);
        const bool inside = tn >= 0 && rel < c.nt;
        const uint32_t bit = (uint32_t)(((uint64_t)tn - p.tile_lo) & 31);
        const uint32_t e1 = p.dir_start[d + 1];
        for (uint32_t e = p.dir_start[d]; e < e1; ++e) {
          const uint32_t j2 = p.link_j2[e];
          uint32_t v = 0;
          if (inside) v = (Z[j2] >> (uint32_t)rel) & 1u;
          else if (tn >= 0) {
            if (e < Epf) v = (S.R[e * kChunkTiles + lane] >> bit) & 1u;
            else v = fetch_cell(cur8, (uint64_t)tn * p.K + j2, p.halo);
          }
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
          if (lane == 0) Z[Kw + e] = bal;
        }
      }
    }
    if (issuer) bulk_wait_read_all();  // Zout(buf) was last stored two chunks ago
    __syncthreads();  // the one CTA barrier per chunk
    if (tid == 0) S.ctr[buf ^ 1] = 0;  // idle: every warp finished the previous chunk's blocks
    if (has_next)
      chunk_neighbours<true>(p, S.ntl, S.R, chunk_info(p, chunk + G), cur8, warp, nwarps, lane);

    // count + rule, one word (32 cells) per lane
    const uint32_t live_lanes = c.nt >= 32 ? 0xFFFFFFFFu : ((1u << c.nt) - 1u);
    const uint8_t* zb = reinterpret_cast<const uint8_t*>(Z);
    uint32_t* out = S.Zout(buf);
    for (uint32_t jb = grab(&S.ctr[buf], lane); jb < nblk; jb = grab(&S.ctr[buf], lane)) {
      const uint32_t j = jb * 32 + lane;
      if (j >= K) continue;
      const uint4 row = __ldg(reinterpret_cast<const uint4*>(p.nbr) + j);  // byte offsets into Z
      uint32_t x[8];
      x[0] = *reinterpret_cast<const uint32_t*>(zb + (row.x & 0xFFFFu));
      x[1] = *reinterpret_cast<const uint32_t*>(zb + (row.x >> 16));
      x[2] = *reinterpret_cast<const uint32_t*>(zb + (row.y & 0xFFFFu));
      x[3] = *reinterpret_cast<const uint32_t*>(zb + (row.y >> 16));
      x[4] = *reinterpret_cast<const uint32_t*>(zb + (row.z & 0xFFFFu));
      if (DMAX > 5) {
        x[5] = *reinterpret_cast<const uint32_t*>(zb + (row.z >> 16));
        x[6] = *reinterpret_cast<const uint32_t*>(zb + (row.w & 0xFFFFu));
        x[7] = *reinterpret_cast<const uint32_t*>(zb + (row.w >> 16));
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
      uint32_t nw;
      if (CONWAY) nw = c1 & ~c2 & ~c3 & (c0 | alive);
      else nw = (alive & rule_bits(p.survive, c0, c1, c2, c3)) | (~alive & rule_bits(p.birth, c0, c1, c2, c3));
      out[j] = nw & live_lanes;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.bar[2 + buf]);
  }
  if (issuer) {  // write out the last chunk
    const int lb = (int)((it - 1) & 1);
    mbar_wait(&S.bar[2 + lb], ((it - 1) >> 1) & 1);
    tma_store_1d(next + (chunk - G) * Kw, S.Zout(lb), cbytes);
    bulk_wait_all();
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------------------------ conversions
// byte layout -> packed: lane = tile reads its 32-byte window (two 128-bit loads), packs, and
// the warp transposes so lane L holds word j0 + my_jj(L).  One warp per (chunk, j-block).
__global__ void k_pack(TileParams p, const uint8_t* __restrict__ st, uint32_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K, nblk = (K + 31) / 32, wpc = (p.Kw + 31) / 32;  // blocks incl. padding words
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);
  const Transposer tr(lane);
  const uint64_t ntiles = p.tile_hi - p.tile_lo;
  for (uint64_t wi = gw; wi < p.nchunks * wpc; wi += nw) {
    const uint64_t c = wi / wpc;
    const uint32_t jb = (uint32_t)(wi - c * wpc), j0 = jb * 32;
    const uint64_t t = c * kChunkTiles + lane;
    uint32_t acc = 0;
    if (jb < nblk && t < ntiles) {
      const uint4* src = reinterpret_cast<const uint4*>(st + t * p.Kp + j0);
      const uint4 lo = __ldg(src), hi = __ldg(src + 1);
      acc = (lo.x & 0x01010101u) | ((lo.y & 0x01010101u) << 1) | ((lo.z & 0x01010101u) << 2) |
            ((lo.w & 0x01010101u) << 3) | ((hi.x & 0x01010101u) << 4) | ((hi.y & 0x01010101u) << 5) |
            ((hi.z & 0x01010101u) << 6) | ((hi.w & 0x01010101u) << 7);
    }
    const uint32_t x = tr(acc);  // bytes past K are zero in the byte layout
    if (j0 + my_jj < p.Kw) packed[c * p.Kw + j0 + my_jj] = x;
  }
}

// packed -> byte layout (every byte of every tile written, padding zero).
__global__ void k_unpack(TileParams p, const uint32_t* __restrict__ packed, uint8_t* __restrict__ st) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K, wpt = p.Kp / 16;  // 16-byte groups per tile
  const uint32_t nblk = (K + 31) / 32;
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);
  const Transposer tr(lane);
  const uint64_t ntiles = p.tile_hi - p.tile_lo;
  const uint32_t jobs = (wpt + 1) / 2;  // 32-byte windows per tile (the last may be 16 bytes)
  for (uint64_t wi = gw; wi < p.nchunks * jobs; wi += nw) {
    const uint64_t c = wi / jobs;
    const uint32_t jb = (uint32_t)(wi - c * jobs), j0 = jb * 32;
    uint32_t x = (jb < nblk && j0 + my_jj < K) ? packed[c * p.Kw + j0 + my_jj] : 0u;
    x = tr(x);
    const uint64_t t = c * kChunkTiles + lane;
    if (t >= ntiles) continue;
    uint4* dst = reinterpret_cast<uint4*>(st + t * p.Kp + j0);
    dst[0] = make_uint4(x & 0x01010101u, (x >> 1) & 0x01010101u, (x >> 2) & 0x01010101u, (x >> 3) & 0x01010101u);
    if (j0 + 16 < p.Kp)
      dst[1] = make_uint4((x >> 4) & 0x01010101u, (x >> 5) & 0x01010101u, (x >> 6) & 0x01010101u,
                          (x >> 7) & 0x01010101u);
  }
}

// D9 initial state straight into the packed layout: lane = tile, one cell per lane, ballot.
__global__ void k_seed_packed(TileParams p, LevelMaps gm, uint32_t* __restrict__ packed, uint64_t mseed, uint64_t q) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x >> 5;
  const uint64_t ntiles = p.tile_hi - p.tile_lo;
  for (uint64_t wi = gw; wi < p.nchunks * p.Kw; wi += nw) {
    const uint64_t c = wi / p.Kw;
    const uint32_t j = (uint32_t)(wi - c * p.Kw);
    const uint64_t t = c * kChunkTiles + lane;
    uint32_t v = 0;
    if (j < p.K && t < ntiles) {
      uint32_t x, y;
      lambda_level(gm, (p.tile_lo + t) * p.K + j, x, y);
      const uint64_t h = [&] {
        uint64_t z = ((((uint64_t)x) << 32) | y) ^ mseed;
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ull;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBull;
        z ^= z >> 31;
        return z;
      }();
      v = (h >> 32) < q ? 1u : 0u;
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
    if (lane == 0) packed[wi] = bal;
  }
}

__global__ void k_count_packed(const uint32_t* __restrict__ w, uint64_t n, unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += __popc(w[i]);
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

// ------------------------------------------------------------------------------------ launchers
using PackedFn = void (*)(TileParams, const uint32_t*, uint32_t*);

static PackedFn pick_packed(const TileParams& p) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  if (p.dmax <= 5) return conway ? k_step_packed<5, true> : k_step_packed<5, false>;
  return conway ? k_step_packed<8, true> : k_step_packed<8, false>;
}

cudaError_t packed_prepare(const TileParams& p, size_t smem, int threads, int* occupancy) {
  PackedFn fn = pick_packed(p);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t launch_step_packed(const TileParams& p, const uint32_t* cur, uint32_t* next, int grid, int threads,
                               size_t smem, cudaStream_t st) {
  if (p.nchunks == 0) return cudaSuccess;
  pick_packed(p)<<<grid, threads, smem, st>>>(p, cur, next);
  return cudaGetLastError();
}

static unsigned warps_grid(uint64_t warps) {
  uint64_t blocks = (warps + 7) / 8;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  return (unsigned)(blocks ? blocks : 1);
}

cudaError_t launch_pack(const TileParams& p, const uint8_t* st, uint32_t* packed, cudaStream_t s) {
  if (p.nchunks == 0) return cudaSuccess;
  k_pack<<<warps_grid(p.nchunks * ((p.Kw + 31) / 32)), 256, 0, s>>>(p, st, packed);
  return cudaGetLastError();
}

cudaError_t launch_unpack(const TileParams& p, const uint32_t* packed, uint8_t* st, cudaStream_t s) {
  if (p.nchunks == 0) return cudaSuccess;
  k_unpack<<<warps_grid(p.nchunks * ((p.Kp / 16 + 1) / 2)), 256, 0, s>>>(p, packed, st);
  return cudaGetLastError();
}

cudaError_t launch_seed_packed(const TileParams& p, const LevelMaps& full, uint32_t* packed, uint64_t seed, uint64_t q,
                               cudaStream_t s) {
  if (p.nchunks == 0) return cudaSuccess;
  uint64_t z = seed;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  k_seed_packed<<<warps_grid(p.nchunks * p.Kw), 256, 0, s>>>(p, full, packed, z, q);
  return cudaGetLastError();
}

cudaError_t launch_count_packed(const uint32_t* w, uint64_t nwords, uint64_t* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (nwords + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_count_packed<<<(unsigned)(blocks ? blocks : 1), 256, 0, s>>>(w, nwords, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

}  // namespace sqz
