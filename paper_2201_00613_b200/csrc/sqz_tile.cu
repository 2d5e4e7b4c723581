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

#include "sqz_bits.cuh"

namespace sqz {

// A chunk is 32 consecutive tiles of Kp bytes, contiguous in HBM and in shared memory (one
// bulk copy each way).  Kp >= round_up(K, 32) (whole 32-byte lane windows) and Kp/16 is odd,
// so the 128-bit accesses of 8 consecutive lanes hit distinct bank groups.
__host__ __device__ inline size_t chunk_buf_bytes(const TileParams& p) { return (size_t)p.Kp * kChunkTiles; }


struct TileSmem {
  uint8_t* in0;    // 2 chunk buffers (input, then output in place)
  uint32_t cb;
  uint32_t* Z0;    // 2 x [K state words | E link words | zero word] (by chunk parity)
  uint32_t zn;
  uint32_t* ntl;   // [ndirs][32] neighbour tile + 1 of each lane's tile (0 = none) — next chunk
  uint32_t* R;     // [E][32] prefetched words holding out-of-chunk neighbour bytes — next chunk
  uint64_t* bar;   // [0,2) TMA loads landed, [2,4) all warps wrote the chunk's output
  uint32_t* ctr;   // [2] Phase-A and [2] count/write-back block counters, by chunk parity
  uint32_t* lj2;   // [E] link e's cell in the neighbour tile, [E, E + ndirs + 1) direction starts
  __device__ __forceinline__ uint8_t* in(int b) const { return in0 + (size_t)b * cb; }
  __device__ __forceinline__ uint32_t* Z(int b) const { return Z0 + (size_t)b * zn; }
};


__host__ __device__ inline size_t tile_layout(const TileParams& p, uint8_t* base, TileSmem* s) {
  size_t off = 0;
  const size_t cb = chunk_buf_bytes(p);
  if (s) {
    s->in0 = base;
    s->cb = (uint32_t)cb;
  }
  off += 2 * cb;
  const size_t zn = align16((size_t)(p.K + p.E + 1) * 4) / 4;
  if (s) {
    s->Z0 = (uint32_t*)(base + off);
    s->zn = (uint32_t)zn;
  }
  off += 2 * zn * 4;
  if (s) s->ntl = (uint32_t*)(base + off);
  off += (size_t)(p.ndirs ? p.ndirs : 1) * kChunkTiles * 4;
  if (s) s->R = (uint32_t*)(base + off);
  off += (size_t)(prefetch_links(p) ? prefetch_links(p) : 1) * kChunkTiles * 4;
  if (s) s->bar = (uint64_t*)(base + off);
  off += 32;
  if (s) s->ctr = (uint32_t*)(base + off);
  off += 16;
  if (s) s->lj2 = (uint32_t*)(base + off);
  off += align16((size_t)(p.E + p.ndirs + 1) * 4);
  return align16(off);
}

size_t tile_smem_bytes(const TileParams& p) { return tile_layout(p, nullptr, nullptr); }

// One thread: the chunk's 32 tiles (nt * Kp contiguous bytes) -> shared memory, one bulk copy.
__device__ __forceinline__ void chunk_load(const TileParams& p, const ChunkInfo& c, uint8_t* buf, uint64_t* bar,
                                           const uint8_t* __restrict__ cur) {
  tma_load_1d(buf, cur + (c.t0 - p.tile_lo) * p.Kp, c.nt * p.Kp, bar);
}

__device__ __forceinline__ void chunk_store(const TileParams& p, const ChunkInfo& c, const uint8_t* buf,
                                            uint8_t* __restrict__ next) {
  tma_store_1d(next + (c.t0 - p.tile_lo) * p.Kp, buf, c.nt * p.Kp);
}

template <int DMAX, bool CONWAY, int MAXT, int MINB, int RB, bool PEER>
__global__ void __launch_bounds__(MAXT, MINB) k_step_tile(TileParams p, const uint8_t* __restrict__ cur,
                                                         uint8_t* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TileSmem S;
  tile_layout(p, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K;
  const uint32_t nblk = (K + 31) / 32;
  const uint32_t Epf = prefetch_links(p);
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);  // cell offset this lane holds after a transpose
  const Transposer tr(lane);
  uint4 rows[RB];  // neighbour-table rows of this lane's static C+D blocks (L1 once per launch)
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t j = ((uint32_t)warp + (uint32_t)(i * nwarps)) * 32 + my_jj;
    rows[i] = j < K ? __ldg(reinterpret_cast<const uint4*>(p.nbr) + j) : make_uint4(0, 0, 0, 0);
  }
  const int lw = nwarps - 1;  // the last warp issues TMA and the coarse λ
  const uint32_t St = p.Kp;   // tile stride in shared memory
  const bool issuer = warp == lw && lane == 0;
  bool peer_sent = false;  // PEER: this lane stored halo cells into a peer buffer

  // the link tables, read every chunk, from shared memory instead of global loads
  for (uint32_t e = tid; e < p.E; e += blockDim.x) S.lj2[e] = p.link_j2[e];
  for (uint32_t d = tid; d <= p.ndirs; d += blockDim.x) S.lj2[p.E + d] = p.dir_start[d];
  if (tid == 0) {
    S.Z(0)[p.zslot] = 0;
    S.Z(1)[p.zslot] = 0;
    S.ctr[0] = S.ctr[1] = S.ctr[2] = S.ctr[3] = 0;
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
  {  // prologue: chunk 0 loaded, neighbours + link prefetch of chunk 0
    const ChunkInfo c0 = chunk_info(p, chunk);
    if (issuer) chunk_load(p, c0, S.in(0), &S.bar[0], cur);
    chunk_neighbours(p, S.ntl, S.R, S.lj2, c0, cur, warp, nwarps, lane);
  }

  uint32_t it = 0;
  for (; chunk < p.nchunks; chunk += G, ++it) {
    const int buf = it & 1;
    const ChunkInfo c = chunk_info(p, chunk);
    const bool has_next = chunk + G < p.nchunks;
    if (has_next) {
      const ChunkInfo cn = chunk_info(p, chunk + G);
      if (issuer) {
        bulk_wait_read_all();  // in(buf^1) held the previous chunk's output
        fence_proxy_async();
        chunk_load(p, cn, S.in(buf ^ 1), &S.bar[buf ^ 1], cur);
      }
    }
    if (tid == 0) S.ctr[buf ^ 1] = 0;  // next chunk's Phase-A counter (idle since the last barrier)
    uint32_t pe0 = 0, pe1 = 0;  // PEER: this chunk's send range, loaded before the compute hides it
    if (PEER && warp == lw) {
      pe0 = p.peer_chunk_start[chunk];
      pe1 = p.peer_chunk_start[chunk + 1];
    }
    mbar_wait(&S.bar[buf], (it >> 1) & 1);
    uint8_t* inb = S.in(buf);
    uint32_t* Zb = S.Z(buf);
    const bool active = (uint32_t)lane < c.nt;

    // Phase B first: boundary-link words; warp w owns the links of directions w, w + nwarps, ...
    // (the same warp computed their neighbour tiles and issued their gathers last iteration).
    // Phase A's blocks are grabbed dynamically afterwards, so warps with heavy link work take fewer.
    if (warp < (int)p.ndirs) {
      cp_async_wait_all();
      for (int d = warp; d < (int)p.ndirs; d += nwarps) {
        const int64_t tn = (int64_t)S.ntl[d * kChunkTiles + lane] - 1;
        const uint64_t rel = (uint64_t)(tn - (int64_t)c.t0);
        const bool inside = tn >= 0 && rel < c.nt;
        const uint32_t e1 = S.lj2[p.E + d + 1];
        for (uint32_t e = S.lj2[p.E + d]; e < e1; ++e) {
          const uint32_t j2 = S.lj2[e];
          uint32_t v = 0;
          if (inside) v = inb[(uint32_t)rel * St + j2];
          else if (tn >= 0) {
            if (e < Epf) v = (S.R[e * kChunkTiles + lane] >> (8 * (j2 & 3u))) & 0xFFu;
            else v = fetch_cell(cur, (uint64_t)tn * p.K + j2, p.halo);
          }
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
          if (lane == 0) Zb[K + e] = bal;
        }
      }
    }
    // Phase A: lane = tile; 32 aligned bytes (cells j0..j0+31 of its slot) -> bits 8p+m =
    // cell 4m+p -> transpose, leaving lane L with the bit-sliced word of cell j0 + my_jj(L)
    const uint32_t in_s = smem_u32(inb) + (uint32_t)lane * St;  // this lane's tile slot
    const uint32_t z_s = smem_u32(Zb);
    const uint32_t ctr_s = smem_u32(&S.ctr[buf]);
    for (uint32_t jb = grab(ctr_s, lane); jb < nblk; jb = grab(ctr_s, lane)) {  // all dynamic
      const uint32_t j0 = jb * 32;
      // Padding bytes (j >= K) and the slots of lanes past a ragged chunk's end only reach
      // words j >= K (not stored) and bit positions of dead tiles (masked at the output).
      const uint32_t x = tr(pack01(lds128(in_s + j0), lds128(in_s + j0 + 16)));
      if (j0 + my_jj < K) sts32(z_s + 4 * (j0 + my_jj), x);
    }
    __syncthreads();  // the one CTA barrier per chunk: all state and link words are in Zb
    // the next chunk's neighbour tiles + link prefetch overlap the count/write-back blocks
    if (has_next) chunk_neighbours(p, S.ntl, S.R, S.lj2, chunk_info(p, chunk + G), cur, warp, nwarps, lane);

    // Phases C + D per j-block: lane L computes cell j0 + my_jj(L) of all 32 tiles (carry-save
    // count, rule), then the block is transposed back (lane = tile) and written in place.
    // Blocks are static (jb = warp + i * nwarps) so the first RB rows of the shared neighbour
    // table stay in registers for the whole launch.
    const uint32_t live_lanes = c.nt >= 32 ? 0xFFFFFFFFu : ((1u << c.nt) - 1u);
    auto block = [&](uint32_t jb, const uint4& row) {
      const uint32_t j0 = jb * 32;
      const uint32_t j = j0 + my_jj;
      uint32_t nw = 0;
      if (j < K) {
        uint32_t x[8];  // slots hold byte offsets into Z
        x[0] = lds32(z_s + (row.x & 0xFFFFu));
        x[1] = lds32(z_s + (row.x >> 16));
        x[2] = lds32(z_s + (row.y & 0xFFFFu));
        x[3] = lds32(z_s + (row.y >> 16));
        x[4] = lds32(z_s + (row.z & 0xFFFFu));
        if (DMAX > 5) {
          x[5] = lds32(z_s + (row.z >> 16));
          x[6] = lds32(z_s + (row.w & 0xFFFFu));
          x[7] = lds32(z_s + (row.w >> 16));
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
        const uint32_t alive = lds32(z_s + 4 * j);
        if (CONWAY) {
          nw = c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23: count 3, or count 2 and alive
        } else {
          nw = (alive & rule_bits(p.survive, c0, c1, c2, c3)) | (~alive & rule_bits(p.birth, c0, c1, c2, c3));
        }
        nw &= live_lanes;
      }
      const uint32_t xb = tr(nw);  // bit 8p+m = cell j0 + 4m + p of this lane's tile (0 past K)
      if (active) {
        const uint32_t m = 0x01010101u;
        sts128(in_s + j0, xb & m, (xb >> 1) & m, (xb >> 2) & m, (xb >> 3) & m);
        sts128(in_s + j0 + 16, (xb >> 4) & m, (xb >> 5) & m, (xb >> 6) & m, (xb >> 7) & m);
      }
    };
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const uint32_t jb = (uint32_t)warp + (uint32_t)(i * nwarps);
      if (jb < nblk) block(jb, rows[i]);
    }
    for (uint32_t jb = (uint32_t)warp + (uint32_t)(RB * nwarps); jb < nblk; jb += (uint32_t)nwarps) {
      const uint32_t j = jb * 32 + my_jj;
      block(jb, j < K ? __ldg(reinterpret_cast<const uint4*>(p.nbr) + j) : make_uint4(0, 0, 0, 0));
    }
    // no CTA barrier: each warp publishes its part of the output; only the storing thread waits
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.bar[2 + buf]);
    if (PEER) {  // the chunk's output complete for the halo epilogue: a named barrier the last warp waits on
      if (warp == lw) asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
      else asm volatile("bar.arrive 1, %0;" ::"r"(blockDim.x) : "memory");
    }
    if (PEER && warp == lw && pe1 > pe0) {
      // fused halo: the last warp stores this chunk's send cells straight into the peers' buffers
      for (uint32_t e = pe0 + (uint32_t)lane; e < pe1; e += 32) {
        const uint32_t cell = p.peer_cell[e];
        p.peer_recv[p.peer_of[e]][p.peer_pos[e]] = inb[(cell >> 16) * St + (cell & 0xFFFFu)];
      }
      peer_sent = true;
      __syncwarp();
    }
    if (issuer) {
      mbar_wait(&S.bar[2 + buf], (it >> 1) & 1);
      chunk_store(p, c, inb, next);
    }
  }
  cp_async_wait_all();
  if (issuer) bulk_wait_all();
  // one system-scope fence per storing thread, not per chunk (a MEMBAR.SYS costs microseconds)
  if (PEER && peer_sent) __threadfence_system();
}

// ---------------------------------------------------------------------------------------

// Tile adjacency (init): one thread per local tile, coarse λ then one coarse ν per direction.
__global__ void k_tile_adjacency(TileParams p, uint32_t* __restrict__ adj) {
  const uint64_t n = p.tile_hi - p.tile_lo;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t X, Y;
    lambda_level(p.coarse, p.tile_lo + i, X, Y);
    for (uint32_t d = 0; d < p.ndirs; ++d) {
      const uint32_t code = (p.dir_code >> (4 * d)) & 0xFu;
      const int dx = (int)(code & 3u) - 1, dy = (int)(code >> 2) - 1;
      const uint64_t nt = nu_level(p.coarse, (int64_t)X + dx, (int64_t)Y + dy);
      adj[d * p.adj_stride + i] = nt == kNoneU64 ? 0u : (uint32_t)(nt + 1);
    }
  }
}

cudaError_t launch_tile_adjacency(const TileParams& p, uint32_t* adj, cudaStream_t st) {
  const uint64_t n = p.tile_hi - p.tile_lo;
  if (n == 0 || p.ndirs == 0) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_tile_adjacency<<<(unsigned)blocks, 256, 0, st>>>(p, adj);
  return cudaGetLastError();
}

using TileFn = void (*)(TileParams, const uint8_t*, uint8_t*);

template <bool PEER>
static TileFn pick_t(const TileParams& p, int threads) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  if (threads <= 256) {
    if (p.dmax <= 5) return conway ? k_step_tile<5, true, 256, 4, 3, PEER> : k_step_tile<5, false, 256, 4, 3, PEER>;
    return conway ? k_step_tile<8, true, 256, 4, 3, PEER> : k_step_tile<8, false, 256, 4, 3, PEER>;
  }
  if (p.dmax <= 5) return conway ? k_step_tile<5, true, 1024, 1, 1, PEER> : k_step_tile<5, false, 1024, 1, 1, PEER>;
  return conway ? k_step_tile<8, true, 1024, 1, 1, PEER> : k_step_tile<8, false, 1024, 1, 1, PEER>;
}

// PEER variants carry the fused peer-memory halo epilogue (sharded contexts with the peer transport).
static TileFn pick(const TileParams& p, int threads) {
  return p.peer_recv ? pick_t<true>(p, threads) : pick_t<false>(p, threads);
}

cudaError_t tile_prepare(const TileParams& p, size_t smem, int threads, int* occupancy) {
  for (TileFn fn : {pick_t<false>(p, threads), pick_t<true>(p, threads)}) {
    cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int blocks = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick_t<false>(p, threads), threads, smem);
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
