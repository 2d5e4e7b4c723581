// sqz_stream.cu — the byte-state step for LARGE tiles.
//
// Link-heavy fractals (the carpet's full tile edges: 112 outside cells per 512-cell tile
// at tile level 3) need larger tiles: at level 4 the carpet's links fall to 328 per 4096 cells
// (SURVEY §7 hard part 3).  A 32-tile chunk of such tiles (131 KB) no longer fits shared memory
// twice, so this kernel keeps only the chunk's bit-sliced form Z (4 B per cell position, bit i =
// tile i, the form k_step_tile builds; double-buffered by chunk parity) and STREAMS the bytes:
//
//   copy thread:  slice q of the chunk (cells [480q, 480q+480) of its 32 tiles) -> input-ring slot
//                 (one 2D TMA box pair on the slot's mbarrier, an L2 prefetch of the slice after)
//   Phase A       slice -> Z (lane = tile: pack 32 bytes, 32x32 warp transpose; slices in pairs)
//   Phase B       boundary-link words by link items: lane = link for the long directions (masked
//                 rotations of the neighbour cell's Z word per in-chunk offset, one gathered word
//                 per outside tile), ballots for the short ones (see link_items)
//   Phase C+D     count + rule per j-block, transpose back, one 256-bit store per lane straight to
//                 HBM; blocks that read no link word before the links barrier
//
// Consumer warp w owns j-block w of every slice (15 warps x 32 cells = 480), so its neighbour
// table rows stay in registers; two named barriers per chunk (Z and gathers complete, link words
// published).  The neighbour structure is the one of k_step_tile (P:57, P:189 at tile level).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "sqz_bits.cuh"

namespace sqz {

constexpr uint32_t kStreamSW = 480;   // cells (bytes) per slice and tile: one j-block per consumer warp
constexpr uint32_t kStreamBox = 240;  // TMA box width: a slice is two [32 tiles x 240 B] boxes; the
                                      // 240-byte row pitch (an odd multiple of 16) keeps the lanes'
                                      // 128-bit accesses (lane = tile) bank-conflict-free
constexpr uint32_t kStreamSlot = 2 * kChunkTiles * kStreamBox;  // bytes per ring slot
constexpr int kStreamNW = 15;         // consumer warps: one j-block of each slice apiece
constexpr int kStreamThreads = 32 * (kStreamNW + 1);
constexpr uint32_t kStreamMaxLinks = 1024;
constexpr uint32_t kStreamMaxItems = 64;  // link groups: ceil(links of d / 32) per direction d

struct StreamSmem {
  uint8_t* in0;     // p.sin slots of two [32][240] boxes
  uint32_t* Z0;     // 2 x [K state words | E link words | zero word], by chunk parity
  uint32_t zn;      // words per Z buffer
  uint32_t* Wn;     // PEER: the chunk's new state words (bit i = tile i), K words
  uint32_t* ntl;    // [2][ndirs][32] neighbour tile + 1 of each lane's tile, by chunk parity
  uint32_t* G;      // [32][E] word holding the neighbour byte of link e for tile i, where tile i's
                    // neighbour tile lies outside the chunk (this chunk's gathers); or COMPACTED
                    // (p.srcap words: only the chunk's outside (tile, link) pairs, see link_prefetch)
  uint32_t* gctr;   // compacted G: [2] words allocated per chunk parity
  uint32_t* grb;    // compacted G: [2][kStreamMaxItems] first word of each group item's gathers
  uint32_t* grbb;   // compacted G: [2][E] first word of each short link's gathers (ballot items)
  uint32_t* lj2;    // [E] link e: its cell in the neighbour tile | direction << 16
  uint32_t* items;  // [kStreamMaxItems] link work items (see link_items)
  uint32_t* nitems;
  uint32_t* slinks; // [E] the links of the short directions, handled by ballots
  uint64_t* bar;    // infull[sin], inempty[sin]
};

__host__ __device__ inline size_t stream_layout(const TileParams& p, bool peer, uint8_t* base, StreamSmem* s) {
  const size_t slot = kStreamSlot;
  size_t off = 0;
  if (s) s->in0 = base + off;
  off += p.sin * slot;
  const size_t zn = align16((size_t)(p.K + p.E + 1) * 4) / 4;
  if (s) {
    s->Z0 = (uint32_t*)(base + off);
    s->zn = (uint32_t)zn;
  }
  off += 2 * zn * 4;
  if (s) s->Wn = (uint32_t*)(base + off);
  off += peer ? align16((size_t)p.K * 4) : 0;
  if (s) s->ntl = (uint32_t*)(base + off);
  off += (size_t)2 * (p.ndirs ? p.ndirs : 1) * kChunkTiles * 4;
  if (s) s->G = (uint32_t*)(base + off);
  off += p.srcap ? align16((size_t)p.srcap * 4) : (size_t)(p.E ? p.E : 1) * kChunkTiles * 4;
  if (s) s->gctr = (uint32_t*)(base + off);
  off += 16;
  if (s) s->grb = (uint32_t*)(base + off);
  off += p.srcap ? (size_t)2 * kStreamMaxItems * 4 : 0;
  if (s) s->grbb = (uint32_t*)(base + off);
  off += p.srcap ? align16((size_t)2 * (p.E ? p.E : 1) * 4) : 0;
  if (s) s->lj2 = (uint32_t*)(base + off);
  off += align16((size_t)(p.E ? p.E : 1) * 4);
  if (s) s->items = (uint32_t*)(base + off);
  off += (size_t)kStreamMaxItems * 4;
  if (s) s->nitems = (uint32_t*)(base + off);
  off += 16;
  if (s) s->slinks = (uint32_t*)(base + off);
  off += align16((size_t)(p.E ? p.E : 1) * 4);
  if (s) s->bar = (uint64_t*)(base + off);
  off += (size_t)2 * p.sin * 8;
  return align16(off);
}

size_t stream_smem_bytes(const TileParams& p, bool peer) { return stream_layout(p, peer, nullptr, nullptr); }

__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(kStreamNW * 32) : "memory");
}

// Shared-memory offset of byte x (a multiple of 16, < 480) of a tile's slice row, relative to the
// row's start in box 0: the row continues in box 1 after 240 bytes.
__device__ __forceinline__ uint32_t box_off(uint32_t x) {
  return x < kStreamBox ? x : x - kStreamBox + kStreamSlot / 2;
}

// 16 warps: 128 registers at one CTA per SM, 64 at two (16K registers per SM sub-partition,
// which holds every fourth warp)
template <int MINB>
struct StreamRegs {
  static constexpr int n = MINB >= 2 ? 64 : 128;
};

// Adjacency words of chunk c (neighbour tile + 1 per link direction and lane tile, built at init)
// -> ntl buffer, by cp.async; warps by direction.  Rows are padded to whole 128-tile chunks.
__device__ __forceinline__ void adj_prefetch(const TileParams& p, uint32_t* ntl, const ChunkInfo& c, int cw, int lane) {
  for (uint32_t d = (uint32_t)cw; d < p.ndirs; d += kStreamNW)
    cp_async4(&ntl[d * kChunkTiles + lane], p.adj + d * p.adj_stride + (c.t0 - p.tile_lo + lane));
  cp_async_commit();
}


// Link work items.  A GROUP item (bit 31 clear: first link | count - 1 << 11 | direction << 16)
// holds up to 32 links of one long direction d (links are sorted by direction); lane = link.
// Tiles of a chunk are lanes of the bit-sliced words, and a direction's neighbour tiles are the same
// for all its links, so per (group, tile) the work is uniform across the warp: the in-chunk part of
// a link word is a few masked rotations of the neighbour cell's Z word (one per distinct lane
// offset rel - i), the out-of-chunk part one gathered word per outside tile.  A BALLOT item (bit 31
// set: first index into slinks | count - 1 << 11) holds the links of the short directions (a
// corner's single link), lane = tile, one ballot per link.  Items are built so that their number
// stays at most one per warp where possible (link_items).
constexpr uint32_t kBallotItem = 1u << 31;
constexpr uint32_t kLongDirection = 8;  // links per direction from which a direction gets group items

__device__ void link_items(const TileParams& p, const StreamSmem& S) {  // one thread, at launch
  uint32_t n = 0, ns = 0;
  for (uint32_t d = 0; d < p.ndirs; ++d) {
    const uint32_t e0 = p.dir_start[d], e1 = p.dir_start[d + 1], nd = e1 - e0;
    if (nd == 0) continue;
    if (nd < kLongDirection) {
      for (uint32_t e = e0; e < e1; ++e) S.slinks[ns++] = e;
      continue;
    }
    const uint32_t ng = (nd + 31) / 32;  // groups of balanced sizes
    for (uint32_t k = 0, e = e0; k < ng; ++k) {
      const uint32_t m = (nd - (e - e0) + (ng - k) - 1) / (ng - k);
      S.items[n++] = e | ((m - 1u) << 11) | (d << 16);
      e += m;
    }
  }
  // the short directions' links in ballot items: as many as the warps left over allow (at least one)
  const uint32_t free_w = n < (uint32_t)kStreamNW ? (uint32_t)kStreamNW - n : 1u;
  const uint32_t nb = ns == 0 ? 0u : min(ns, free_w);
  for (uint32_t k = 0, i = 0; k < nb; ++k) {
    const uint32_t m = (ns - i + (nb - k) - 1) / (nb - k);
    S.items[n++] = kBallotItem | i | ((m - 1u) << 11);
    i += m;
  }
  *S.nitems = n;
}

struct LinkGroup {
  uint32_t e;      // this lane's link (valid lanes: lane < n)
  uint32_t j2;     // its cell in the neighbour tile
  uint32_t d;      // direction
  bool valid;
};

__device__ __forceinline__ LinkGroup link_group(const StreamSmem& S, uint32_t item, int lane) {
  LinkGroup g;
  const uint32_t e0 = item & 0x7FFu, n = ((item >> 11) & 31u) + 1u;
  g.d = (item >> 16) & 0xFFu;
  g.valid = (uint32_t)lane < n;
  g.e = e0 + (g.valid ? (uint32_t)lane : 0u);
  g.j2 = S.lj2[g.e] & 0xFFFFu;
  return g;
}

// The word holding byte j2 of local tile tl (its 4-byte group), or for another shard's tile the
// cell from the halo placed at its byte: a compacted G's overflow, read synchronously.
__device__ __forceinline__ uint32_t stream_gather(const TileParams& p, const uint8_t* __restrict__ cur, uint32_t tl,
                                                  uint32_t j2, uint32_t nloc) {
  if (tl >= nloc) return fetch_cell(cur, (uint64_t)(tl + (uint32_t)p.tile_lo) * p.K + j2, p.halo) << (8 * (j2 & 3u));
  return __ldg(reinterpret_cast<const uint32_t*>(cur + (uint64_t)tl * p.Kp + (j2 & ~3u)));
}

// Item k = warp cw, cw + NW, ...: for every tile i of chunk c whose neighbour tile in the item's
// direction lies outside the chunk, the 4-byte word holding the neighbour cell of each of the
// item's links, into G[i][e], by cp.async (or, for another shard's tile, from the halo).  The
// same warp consumes them in Phase B of chunk c.  Tile indices fit 32 bits (checked on the host).
// COMPACTED G (p.srcap != 0, link-heavy tiles at two CTAs per SM): only the chunk's (outside tile,
// link) pairs get a word; each item takes its words with one shared atomicAdd on the chunk parity's
// counter and records where they start (grb / grbb), the words of its r-th outside tile (ballot
// order) being base + r n + link (group items) or base + rank of the tile (ballot items); pairs past
// srcap are read synchronously by link_words (stream_gather).
__device__ __forceinline__ void link_prefetch(const TileParams& p, const StreamSmem& S, const uint32_t* ntl,
                                              const ChunkInfo& c, const uint8_t* __restrict__ cur, int cw, int lane,
                                              uint32_t par) {
  const uint32_t t0 = (uint32_t)c.t0, tlo = (uint32_t)p.tile_lo, nloc = (uint32_t)(p.tile_hi - p.tile_lo);
  const uint32_t ni = *S.nitems, E = p.E, cap = p.srcap, lt = (1u << lane) - 1u;
  for (uint32_t k = (uint32_t)cw; k < ni; k += kStreamNW) {
    const uint32_t item = S.items[k];
    if (item & kBallotItem) {  // lane = tile, link by link
      const uint32_t i0 = item & 0x7FFu, n = ((item >> 11) & 31u) + 1u;
      for (uint32_t i = i0; i < i0 + n; ++i) {
        const uint32_t e = S.slinks[i], le = S.lj2[e], j2 = le & 0xFFFFu;
        const uint32_t a1 = ntl[(le >> 16) * kChunkTiles + lane];
        const uint32_t tl = a1 - 1u - tlo;
        const bool out = a1 != 0u && a1 - 1u - t0 >= c.nt;
        uint32_t slot = (uint32_t)lane * E + e;
        bool fits = true;
        if (cap) {
          const uint32_t om = __ballot_sync(0xFFFFFFFFu, out);
          uint32_t base = 0;
          if (lane == 0 && om) base = atomicAdd(&S.gctr[par], (uint32_t)__popc(om));
          base = __shfl_sync(0xFFFFFFFFu, base, 0);
          if (lane == 0) S.grbb[par * E + i] = base;
          slot = base + (uint32_t)__popc(om & lt);
          fits = slot < cap;
        }
        if (out && fits && tl >= nloc) S.G[slot] = fetch_cell(cur, (uint64_t)(a1 - 1u) * p.K + j2, p.halo) << (8 * (j2 & 3u));
        else cp_async4_if(smem_u32(S.G) + 4u * (fits ? slot : 0u), cur + (uint64_t)(out ? tl : 0u) * p.Kp + (j2 & ~3u),
                          out && fits ? 1u : 0u);
      }
      continue;
    }
    const LinkGroup g = link_group(S, item, lane);
    const uint32_t a1 = ntl[g.d * kChunkTiles + lane];  // lane = tile here: neighbour tile + 1 (0 = none)
    const uint32_t tl = a1 - 1u - tlo;
    const bool out = a1 != 0u && a1 - 1u - t0 >= c.nt;
    uint32_t om = __ballot_sync(0xFFFFFFFFu, out);
    const uint32_t farm = __ballot_sync(0xFFFFFFFFu, out && tl >= nloc);  // outside this shard: the halo
    const uint32_t n = ((item >> 11) & 31u) + 1u, jo = g.j2 & ~3u, pv = g.valid ? 1u : 0u;
    uint32_t br = 0;  // compacted: first word of the current outside tile's n links
    if (cap) {
      const uint32_t cnt = (uint32_t)__popc(om) * n;
      if (lane == 0 && cnt) br = atomicAdd(&S.gctr[par], cnt);
      br = __shfl_sync(0xFFFFFFFFu, br, 0);
      if (lane == 0) S.grb[par * kStreamMaxItems + k] = br;
    }
    const uint32_t gs = smem_u32(S.G) + 4u * g.e;
    while (om) {
      const uint32_t i = __ffs(om) - 1u;
      om &= om - 1u;
      const uint32_t tli = __shfl_sync(0xFFFFFFFFu, tl, i);
      const uint32_t dst = cap ? smem_u32(S.G) + 4u * (br + (uint32_t)lane) : gs + i * (E * 4u);
      const uint32_t ok = cap ? (br + n <= cap ? pv : 0u) : pv;
      br += n;
      if (!((farm >> i) & 1u)) {
        cp_async4_if(ok ? dst : smem_u32(S.G), cur + (uint64_t)tli * p.Kp + jo, ok);
      } else if (ok) {  // another shard's tile (sharded contexts): rare, synchronous
        sts32(dst, fetch_cell(cur, (uint64_t)(tli + tlo) * p.K + g.j2, p.halo) << (8 * (g.j2 & 3u)));
      }
    }
  }
  cp_async_commit();
}

// Phase B for item k of chunk c: link word e (bit i = neighbour cell of tile i) -> Z[K + e].
__device__ __forceinline__ void link_words(const TileParams& p, const StreamSmem& S, uint32_t* Z,
                                           const uint32_t* ntl, const ChunkInfo& c, const uint8_t* __restrict__ cur,
                                           int cw, int lane, uint32_t par) {
  const uint32_t t0 = (uint32_t)c.t0, ni = *S.nitems, E = p.E, K = (uint32_t)p.K, cap = p.srcap;
  const uint32_t tlo = (uint32_t)p.tile_lo, nloc = (uint32_t)(p.tile_hi - p.tile_lo), lt = (1u << lane) - 1u;
  for (uint32_t k = (uint32_t)cw; k < ni; k += kStreamNW) {
    const uint32_t item = S.items[k];
    if (item & kBallotItem) {  // lane = tile, one ballot per link
      const uint32_t i0 = item & 0x7FFu, n = ((item >> 11) & 31u) + 1u;
      for (uint32_t i = i0; i < i0 + n; ++i) {
        const uint32_t e = S.slinks[i], le = S.lj2[e], j2 = le & 0xFFFFu;
        const uint32_t a1 = ntl[(le >> 16) * kChunkTiles + lane];
        const uint32_t rel = a1 - 1u - t0;
        const bool inside = a1 != 0u && rel < c.nt;
        uint32_t gw = 0;
        if (cap) {
          const uint32_t om = __ballot_sync(0xFFFFFFFFu, a1 != 0u && !inside);
          const uint32_t slot = S.grbb[par * E + i] + (uint32_t)__popc(om & lt);
          if (a1 != 0u && !inside) gw = slot < cap ? S.G[slot] : stream_gather(p, cur, a1 - 1u - tlo, j2, nloc);
        } else if (a1 != 0u && !inside) {
          gw = S.G[lane * E + e];
        }
        const uint32_t v = inside ? Z[j2] >> (rel & 31u) : gw >> (8u * (j2 & 3u));
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v & 1u);
        if (lane == 0) Z[K + e] = bal;
      }
      continue;
    }
    const LinkGroup g = link_group(S, item, lane);
    const uint32_t a1 = ntl[g.d * kChunkTiles + lane];  // lane = tile
    const uint32_t rel = a1 - 1u - t0;
    const bool present = a1 != 0u, inside = present && rel < c.nt;
    const uint32_t dl = (rel - (uint32_t)lane) & 31u;  // tile i's neighbour is tile i + dl (mod 32)
    uint32_t im = __ballot_sync(0xFFFFFFFFu, inside);
    uint32_t om = __ballot_sync(0xFFFFFFFFu, present && !inside);
    const uint32_t z = Z[g.j2];  // lane = link from here on
    uint32_t w = 0;
    while (im) {  // tiles with the same offset: one masked rotation
      const uint32_t dd = __shfl_sync(0xFFFFFFFFu, dl, __ffs(im) - 1u);
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, inside && dl == dd);
      im &= ~m;
      w |= __funnelshift_r(z, z, dd) & m;
    }
    const uint32_t sh = 8u * (g.j2 & 3u);
    if (cap) {  // compacted: the gathered words in the prefetch's order
      const uint32_t n = ((item >> 11) & 31u) + 1u, tl = a1 - 1u - tlo;
      uint32_t br = S.grb[par * kStreamMaxItems + k];
      while (om) {
        const uint32_t i = __ffs(om) - 1u;
        om &= om - 1u;
        const uint32_t tli = __shfl_sync(0xFFFFFFFFu, tl, i);
        const uint32_t gv = !g.valid ? 0u : br + n <= cap ? S.G[br + lane] : stream_gather(p, cur, tli, g.j2, nloc);
        br += n;
        w |= ((gv >> sh) & 1u) << i;
      }
    }
    const uint32_t gs = smem_u32(S.G) + 4u * g.e;
    while (om) {  // tiles whose neighbour tile is outside the chunk: the gathered words, two at a time
      const uint32_t i = __ffs(om) - 1u;
      om &= om - 1u;
      const uint32_t i2 = om ? __ffs(om) - 1u : i;
      om &= om - 1u;
      const uint32_t g1 = g.valid ? lds32(gs + i * (E * 4u)) : 0u, g2 = g.valid ? lds32(gs + i2 * (E * 4u)) : 0u;
      w |= (((g1 >> sh) & 1u) << i) | (((g2 >> sh) & 1u) << i2);
    }
    if (g.valid) Z[K + g.e] = w;
  }
}

// 32 bytes to global memory with one 256-bit store (32-byte aligned).
__device__ __forceinline__ void stg256(void* dst, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t a4,
                                       uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(a0), "r"(a1), "r"(a2),
               "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
               : "memory");
}

template <int DMAX, bool CONWAY, int RB, int MINB, int NIN, bool PEER>
__global__ void __maxnreg__(StreamRegs<MINB>::n) k_step_stream(TileParams p, const uint8_t* __restrict__ cur,
                                                              uint8_t* __restrict__ next,
                                                              const __grid_constant__ CUtensorMap tm_in) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  StreamSmem S;
  stream_layout(p, PEER, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t K = (uint32_t)p.K, Kp = p.Kp, E = p.E;
  const uint32_t KP32 = (K + 31) & ~31u, nblk = KP32 / 32;
  const uint32_t nsl = (KP32 + kStreamSW - 1) / kStreamSW;
  uint64_t* infull = S.bar;
  uint64_t* inempty = S.bar + NIN;

  for (uint32_t e = tid; e < E; e += blockDim.x) S.lj2[e] = p.link_j2[e] | ((uint32_t)p.link_dir[e] << 16);
  if (tid == 0) {
    S.gctr[0] = S.gctr[1] = 0;
    link_items(p, S);
    S.Z0[p.zslot] = 0;
    S.Z0[S.zn + p.zslot] = 0;
    for (uint32_t i = 0; i < NIN; ++i) {
      mbar_init(&infull[i], 1);
      mbar_init(&inempty[i], kStreamNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if ((uint64_t)blockIdx.x >= p.nchunks) return;
  const uint64_t G = gridDim.x;
  const uint32_t in_base = smem_u32(S.in0);
  const uint32_t slot_bytes = kStreamSlot;

  if (warp == 0) {  // ------------------------------------------- the copy warp (one thread): slices in
    if (lane == 0) {
      const uint32_t total = (uint32_t)((p.nchunks - blockIdx.x + G - 1) / G) * nsl;
      auto load = [&](uint32_t s) {  // slice s of this CTA: two 2D boxes [32 tiles x 240 B] (rows past the
        const uint32_t slot = s % NIN, q = s % nsl;  // shard and columns past round_up(K, 32) read as zero)
        const uint64_t chunk = blockIdx.x + (uint64_t)(s / nsl) * G;
        const uint32_t bar = smem_u32(&infull[slot]);
        const int32_t row = (int32_t)(chunk * kChunkTiles), x0 = (int32_t)(q * kStreamSW);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kStreamSlot) : "memory");
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
              "[%4];" ::"r"(in_base + slot * slot_bytes + h * (kStreamSlot / 2)),
              "l"(&tm_in), "r"(x0 + h * (int32_t)kStreamBox), "r"(row), "r"(bar)
              : "memory");
      };
      auto prefetch = [&](uint32_t s) {  // slice s into L2 (the slice after the one just issued: the next
        const uint32_t q = s % nsl;      // chunk's last slice otherwise waits for its slot at full latency)
        const int32_t row = (int32_t)((blockIdx.x + (uint64_t)(s / nsl) * G) * kChunkTiles), x0 = (int32_t)(q * kStreamSW);
        for (int h = 0; h < 2; ++h)
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&tm_in),
                       "r"(x0 + h * (int32_t)kStreamBox), "r"(row)
                       : "memory");
      };
      uint32_t ld = 0;
      for (; ld < NIN && ld < total; ++ld) load(ld);
      if (ld < total) prefetch(ld);
      // Phase A frees the input slots one slice at a time; each freed slot takes the slice NIN ahead
      for (; ld < total; ++ld) {
        mbar_wait(&inempty[ld % NIN], ((ld - NIN) / NIN) & 1);
        load(ld);
        if (ld + 1 < total) prefetch(ld + 1);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int cw = warp - 1;
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);  // cell offset this lane holds after a transpose
  const Transposer tr(lane);
  uint4 rows[RB];  // neighbour-table rows of this warp's j-blocks (block cw of slices 0..RB-1)
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t j = ((uint32_t)i * kStreamNW + (uint32_t)cw) * 32 + my_jj;
    rows[i] = j < K ? __ldg(reinterpret_cast<const uint4*>(p.nbr) + j) : make_uint4(0, 0, 0, 0);
  }
  // slices q < RB whose block reads a link word (a neighbour slot in [K, K + E)): done after the
  // link words are published; link-free blocks first, so early warps overlap the link phase
  uint32_t lmask = 0;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t lo = 4u * K, hi = 4u * (K + E);
    const uint4 r = rows[i];
    const uint32_t v[8] = {r.x & 0xFFFFu, r.x >> 16, r.y & 0xFFFFu, r.y >> 16,
                           r.z & 0xFFFFu, r.z >> 16, r.w & 0xFFFFu, r.w >> 16};
    bool dep = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) dep |= v[k] >= lo && v[k] < hi;
    if (__any_sync(0xFFFFFFFFu, dep)) lmask |= 1u << i;
  }
  const uint32_t ntl_words = (p.ndirs ? p.ndirs : 1) * kChunkTiles;
  bool peer_sent = false;
  // Phase A per-lane constants (opaque, so ptxas keeps them instead of re-deriving them per slice):
  // the lane's two 16-byte units of its warp's j-block in slot 0, and its cell within a slice
  const uint32_t ja = (uint32_t)cw * 32, jl = ja + my_jj, za = opaque_u32(4 * jl);
  const uint32_t na = opaque_u32(KP32 > ja ? KP32 - ja : 0u), nl = opaque_u32(K > jl ? K - jl : 0u);
  const uint32_t pa0 = opaque_u32(in_base + (uint32_t)lane * kStreamBox + box_off(ja));
  const uint32_t pa1 = opaque_u32(in_base + (uint32_t)lane * kStreamBox + box_off(ja + 16));
  {  // prologue: adjacency of the first two chunks, the first chunk's link gathers
    adj_prefetch(p, S.ntl, chunk_info(p, blockIdx.x), cw, lane);
    if (blockIdx.x + G < p.nchunks) adj_prefetch(p, S.ntl + ntl_words, chunk_info(p, blockIdx.x + G), cw, lane);
    cp_async_wait_all();
    consumers_sync();
    link_prefetch(p, S, S.ntl, chunk_info(p, blockIdx.x), cur, cw, lane, 0u);
  }

  uint32_t seq = 0, it = 0;
  for (uint64_t chunk = blockIdx.x; chunk < p.nchunks; chunk += G, seq += nsl, ++it) {
    const ChunkInfo c = chunk_info(p, chunk);
    if (cw == 0 && lane == 0) S.gctr[(it + 1) & 1u] = 0;  // compacted G: chunk it+1's prefetch allocates from it
    uint32_t* ntl = S.ntl + (it & 1) * ntl_words;
    uint32_t* Zb = S.Z0 + (it & 1) * S.zn;  // double-buffered: no barrier between C+D and the next Phase A
    const uint32_t z_s = smem_u32(Zb);
    uint32_t pe0 = 0, pe1 = 0;
    if (PEER && cw == kStreamNW - 1) {
      pe0 = p.peer_chunk_start[chunk];
      pe1 = p.peer_chunk_start[chunk + 1];
    }
    // Phase A: slice q, j-block q * NW + cw -> Z
    // Slices in pairs: two independent transpose chains per warp interleave (the shuffle chain's
    // latency, not its instruction count, bounds this phase at 16 warps per SM)
    uint32_t q = 0, qc = 0, zq = z_s + za;
    for (; MINB == 1 && q + 1 < nsl; q += 2, qc += 2 * kStreamSW, zq += 8 * kStreamSW) {  // (64 registers: singles)
      const uint32_t s0 = seq + q, s1 = s0 + 1, slot0 = s0 % NIN, slot1 = s1 % NIN;
      mbar_wait(&infull[slot0], (s0 / NIN) & 1);
      mbar_wait(&infull[slot1], (s1 / NIN) & 1);
      const uint4 l0 = lds128(pa0 + slot0 * slot_bytes), h0 = lds128(pa1 + slot0 * slot_bytes);
      const uint4 l1 = lds128(pa0 + slot1 * slot_bytes), h1 = lds128(pa1 + slot1 * slot_bytes);
      const uint32_t x0 = tr(pack01(l0, h0)), x1 = tr(pack01(l1, h1));  // (past K: not stored)
      if (qc < nl) sts32(zq, x0);  // cell j < K
      if (qc + kStreamSW < nl) sts32(zq + 4 * kStreamSW, x1);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&inempty[slot0]);
        mbar_arrive(&inempty[slot1]);
      }
    }
    for (; q < nsl; ++q, qc += kStreamSW, zq += 4 * kStreamSW) {  // an odd last slice
      const uint32_t s = seq + q, slot = s % NIN;
      mbar_wait(&infull[slot], (s / NIN) & 1);
      if (qc < na) {  // this warp's j-block exists in slice q
        const uint32_t x = tr(pack01(lds128(pa0 + slot * slot_bytes), lds128(pa1 + slot * slot_bytes)));
        if (qc < nl) sts32(zq, x);  // cell j < K
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&inempty[slot]);
    }
    cp_async_wait_all();  // this chunk's link gathers and the next chunk's adjacency (own copies)
    consumers_sync();     // Z, R and both adjacency buffers visible to every consumer warp

    // Phase B: link words, by link groups (lane = link)
    link_words(p, S, Zb, ntl, c, cur, cw, lane, it & 1u);

    // Phase C+D: j-block q * NW + cw -> HBM (lane = tile: one 256-bit store of its 32 cells)
    const uint32_t live_lanes = c.nt >= 32 ? 0xFFFFFFFFu : ((1u << c.nt) - 1u);
    uint8_t* tile_out = next + (uint64_t)((uint32_t)(c.t0 - p.tile_lo) + (uint32_t)lane) * Kp;
    const uint32_t zA = z_s + za;  // Z word of this lane's cell in slice 0
    uint8_t* const outA = tile_out + ja;
    // the new state word of this lane's cell in the block at offset qc (0 for cells past K)
    auto block_nw = [&](uint32_t qc, const uint4& row) -> uint32_t {
      uint32_t nw = 0;
      if (qc < nl) {  // cell j < K
        uint32_t x[8];
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
        const uint32_t alive = lds32(zA + 4 * qc);
        if (CONWAY) nw = c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23
        else nw = (alive & rule_bits(p.survive, c0, c1, c2, c3)) | (~alive & rule_bits(p.birth, c0, c1, c2, c3));
        nw &= live_lanes;
        if (PEER) S.Wn[jl + qc] = nw;
      }
      return nw;
    };
    // xb: the transposed block, bit 8p+m = cell 4m+p of the block in this lane's tile (0 past K)
    auto block_out = [&](uint32_t qc, uint32_t xb) {
      const uint32_t m = 0x01010101u;
      if (qc < na && (uint32_t)lane < c.nt)  // Kp = round_up(K, 32): the block's 32 bytes are one sector
        stg256(outA + qc, xb & m, (xb >> 1) & m, (xb >> 2) & m, (xb >> 3) & m, (xb >> 4) & m, (xb >> 5) & m,
               (xb >> 6) & m, (xb >> 7) & m);
    };
    // qc: the block's cell offset from this warp's block of slice 0 (q * NW * 32 unless rotated)
    auto slice_out = [&](uint32_t qc, const uint4& row) {
      if (qc < na) block_out(qc, tr(block_nw(qc, row)));  // this warp's j-block exists in slice q
    };
    auto pair_out = [&](uint32_t qa, const uint4& ra, uint32_t qb, const uint4& rb) {  // two chains interleave
      const uint32_t wa = block_nw(qa, ra), wb = block_nw(qb, rb);
      const uint32_t xa = tr(wa), xb = tr(wb);
      block_out(qa, xa);
      block_out(qb, xb);
    };
    constexpr int RP = MINB == 1 ? RB / 2 : 0;  // block pairs at one CTA per SM (128 registers)
#pragma unroll
    for (int i = 0; i < RP; ++i)  // link-free pairs
      if ((uint32_t)(2 * i + 1) < nsl && !((lmask >> (2 * i)) & 3u))
        pair_out((uint32_t)(2 * i) * kStreamSW, rows[2 * i], (uint32_t)(2 * i + 1) * kStreamSW, rows[2 * i + 1]);
#pragma unroll
    for (int i = 2 * RP; i < RB; ++i)  // link-free single blocks
      if ((uint32_t)i < nsl && !((lmask >> i) & 1u)) slice_out((uint32_t)i * kStreamSW, rows[i]);
    consumers_sync();  // link words published; G and this chunk's adjacency buffer are free
    // slices q >= RB read their neighbour-table rows through L1, one slice ahead (the first one now)
    // so the load latency is hidden.  A partial last slice (r < NW blocks) goes to the LAST r warps
    // here (Phase A gave it to the first r), so every warp carries the same number of blocks per chunk.
    auto tail_block = [&](uint32_t q, uint32_t& qc) -> bool {  // false: no block of this warp in slice q
      const uint32_t r = nblk - q * kStreamNW, sh = q + 1 == nsl && r < kStreamNW ? kStreamNW - r : 0u;
      qc = q * kStreamSW - sh * 32;
      return (uint32_t)cw >= sh;
    };
    // (one CTA per SM only: at two, 64 registers, the live row spills: bottles 0.85 -> 0.90 ms)
    auto tail_row = [&](uint32_t q) -> uint4 {
      uint32_t qc;
      if (q >= nsl || !tail_block(q, qc) || jl + qc >= K) return make_uint4(0, 0, 0, 0);
      return __ldg(reinterpret_cast<const uint4*>(p.nbr) + jl + qc);
    };
    uint4 rown = make_uint4(0, 0, 0, 0);
    if (MINB == 1) rown = tail_row(RB);
    if (chunk + 2 * G < p.nchunks) adj_prefetch(p, ntl, chunk_info(p, chunk + 2 * G), cw, lane);
    if (chunk + G < p.nchunks)
      link_prefetch(p, S, S.ntl + ((it + 1) & 1) * ntl_words, chunk_info(p, chunk + G), cur, cw, lane, (it + 1) & 1u);
#pragma unroll
    for (int i = 0; i < RP; ++i) {  // pairs reading link words (or a pair past the chunk's slices)
      if ((uint32_t)(2 * i + 1) < nsl) {
        if ((lmask >> (2 * i)) & 3u)
          pair_out((uint32_t)(2 * i) * kStreamSW, rows[2 * i], (uint32_t)(2 * i + 1) * kStreamSW, rows[2 * i + 1]);
      } else if ((uint32_t)(2 * i) < nsl) {
        slice_out((uint32_t)(2 * i) * kStreamSW, rows[2 * i]);
      }
    }
#pragma unroll
    for (int i = 2 * RP; i < RB; ++i)  // single blocks reading link words
      if ((uint32_t)i < nsl && ((lmask >> i) & 1u)) slice_out((uint32_t)i * kStreamSW, rows[i]);
    for (uint32_t q = RB; q < nsl; ++q) {
      uint32_t qc;
      const bool mine = tail_block(q, qc);
      if (MINB == 1) {
        const uint4 row = rown;
        rown = tail_row(q + 1);
        if (mine) slice_out(qc, row);
      } else if (mine) {
        slice_out(qc, tail_row(q));
      }
    }
    if (PEER) consumers_sync();  // the chunk's new state words Wn complete for the halo epilogue
    if (PEER && cw == kStreamNW - 1 && pe1 > pe0) {
      // fused halo: the chunk's send cells, from the new state words, straight into the peers' buffers
      for (uint32_t e = pe0 + (uint32_t)lane; e < pe1; e += 32) {
        const uint32_t cell = p.peer_cell[e];
        p.peer_recv[p.peer_of[e]][p.peer_pos[e]] = (uint8_t)((S.Wn[cell & 0xFFFFu] >> (cell >> 16)) & 1u);
      }
      peer_sent = true;
    }
  }
  cp_async_wait_all();
  if (PEER && peer_sent) __threadfence_system();
}

using StreamFn = void (*)(TileParams, const uint8_t*, uint8_t*, const CUtensorMap);

template <bool PEER, int RB, int MINB, int NIN>
static StreamFn pick_stream_r(const TileParams& p) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  if (p.dmax <= 5)
    return conway ? k_step_stream<5, true, RB, MINB, NIN, PEER> : k_step_stream<5, false, RB, MINB, NIN, PEER>;
  return conway ? k_step_stream<8, true, RB, MINB, NIN, PEER> : k_step_stream<8, false, RB, MINB, NIN, PEER>;
}

// RB = slices whose neighbour rows stay in registers: 8 at one CTA per SM (carpet level 4: 8 of
// its 9 slices), 1 at two CTAs per SM (64 registers; empty bottles level 4: 0.82 ms against 0.90
// with 2, which spills).
template <bool PEER>
static StreamFn pick_stream_t(const TileParams& p, int minb) {
  if (minb >= 2) return pick_stream_r<PEER, 1, 2, 4>(p);
  return p.sin >= 8 ? pick_stream_r<PEER, 8, 1, 8>(p) : pick_stream_r<PEER, 8, 1, 4>(p);
}

// The input ring depth p.sin (a power of two: slot indices are masks) and CTAs per SM: two CTAs
// per SM with 4 slots each when that fits twice, else one CTA with 8 slots (the whole next chunk of
// a level-4 carpet but one slice in flight while the current one is computed), else 4.
bool stream_plan(TileParams& p, bool peer, int* minb) {
  if (p.E > kStreamMaxLinks) return false;
  // one CTA per SM: 227 KB; two: 113 KB each (228 KB per SM, 1 KB of it reserved per CTA)
  const size_t cap = 227 * 1024, cap2 = 113 * 1024;
  const char* force = getenv("SQZ_STREAM_CTAS");  // tuning knob: 1 or 2 CTAs per SM
  p.sin = 4;
  p.srcap = 0;
  if ((!force || atoi(force) >= 2) && stream_smem_bytes(p, peer) <= cap2) {
    *minb = 2;
    return true;
  }
  // link-heavy tiles (the carpet at level 4: [32][328] gather words = 42 KB) can run two CTAs per
  // SM with the COMPACTED gather buffer (the chunk's outside (tile, link) pairs, at most ~2K words
  // for the carpet), if it leaves room for the outside pairs of 4 tiles per link.  Opt-in: the
  // carpet runs faster at one CTA per SM with 128 registers (0.515 against 0.523 ms; the full
  // square at level 6 the other way round, 0.0474 against 0.0436 ms; profiles/ab/round2_stream_*)
  const char* compact = getenv("SQZ_STREAM_COMPACT");  // tuning knob: 1 = two CTAs with compacted gathers
  if ((!force || atoi(force) >= 2) && compact && atoi(compact) != 0) {
    p.srcap = 32;
    const size_t base = stream_smem_bytes(p, peer) - 32 * 4;
    if (base < cap2) {
      p.srcap = (uint32_t)((cap2 - base) / 4) & ~31u;
      const char* rc = getenv("SQZ_STREAM_RCAP");  // tests: a smaller buffer (overflow read synchronously)
      const uint32_t want = rc ? (uint32_t)atoi(rc) : 0u;
      if (p.srcap >= 4 * p.E && stream_smem_bytes(p, peer) <= cap2) {
        if (want) p.srcap = std::min(p.srcap, std::max(32u, want & ~31u));
        *minb = 2;
        return true;
      }
    }
    p.srcap = 0;
  }
  *minb = 1;
  p.sin = 8;
  if (stream_smem_bytes(p, peer) <= cap) return true;
  p.sin = 4;
  return stream_smem_bytes(p, peer) <= cap;
}

int stream_threads() { return kStreamThreads; }

cudaError_t stream_prepare(const TileParams& p, size_t smem, int minb, int* occupancy) {
  for (StreamFn fn : {pick_stream_t<false>(p, minb), pick_stream_t<true>(p, minb)}) {
    cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int blocks = 0;
  cudaError_t e =
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick_stream_t<false>(p, minb), kStreamThreads, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

// 2D tensor map of a tile-padded state buffer (streaming contexts: Kp = round_up(K, 32)): dim 0 = the
// Kp bytes of a tile, dim 1 = the shard's tiles; boxes of [32 tiles x 240 B]; out-of-range reads
// are zero.
static cudaError_t state_tensor_map(CUtensorMap* tm, const TileParams& p, const void* base) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {p.Kp, p.tile_hi - p.tile_lo};
  const cuuint64_t strides[1] = {p.Kp};
  const cuuint32_t box[2] = {kStreamBox, kChunkTiles};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_step_stream(const TileParams& p, const uint8_t* cur, uint8_t* next, int grid, int minb,
                               size_t smem, cudaStream_t st) {
  if (p.nchunks == 0) return cudaSuccess;
  // 256-bit stores of whole 32-cell blocks: rows of Kp = round_up(K, 32) bytes, 32-byte aligned buffers
  if (p.Kp != ((p.K + 31) & ~31ull) || ((uintptr_t)cur & 31u) || ((uintptr_t)next & 31u)) return cudaErrorInvalidValue;
  alignas(64) CUtensorMap tin;
  cudaError_t e = state_tensor_map(&tin, p, cur);
  if (e != cudaSuccess) return e;
  StreamFn fn = p.peer_recv ? pick_stream_t<true>(p, minb) : pick_stream_t<false>(p, minb);
  fn<<<grid, kStreamThreads, smem, st>>>(p, cur, next, tin);
  return cudaGetLastError();
}

}  // namespace sqz
