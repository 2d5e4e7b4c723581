// sqz_packed.cu — the automaton step on the BIT-SLICED PACKED state.
//
// Packed layout (include/squeeze.h): the shard's level-g tiles in chunks of kPackTiles = 128
// consecutive tiles; chunk c holds Kw = round_up(K, 4) 128-bit words; u32 lane q of word j,
// bit i = cell j of tile 128c + 32q + i.  It is the bit-sliced form the byte-state kernel
// (sqz_tile.cu) builds in shared memory, four 32-tile slices side by side, so a step is:
// bulk-copy the chunk's words in, add one word per tile-boundary link, carry-save count + rule
// per word (one 128-bit word = 128 cells per lane), store the words.  1 bit per cell in HBM
// (0.25 B of traffic per cell per step instead of 2 B) and no byte<->bit staging.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "sqz_bits.cuh"

namespace sqz {

// ------------------------------------------------------------------------------------ layout
// CTA work unit = one chunk.  Two rings of bulk copies, each with its own mbarriers:
//  * state stages (p.pstages): [Kw state words (TMA target) | E link words | zero word], 16 B
//    each; chunk i+pstages-1 is issued when chunk i's barrier frees the stage of chunk i-1;
//  * adjacency slots (kAdjSlots): the chunk's rows of the tile adjacency table (128 words per
//    link direction), issued kAdjSlots-1 chunks ahead, so the out-of-chunk link gathers of the
//    next chunk never wait for its state copy.
// Results go straight from registers to HBM (coalesced 512-byte warp stores): no output staging
// and one CTA barrier per chunk.
constexpr uint32_t kAdjSlots = 4;
constexpr uint32_t kPackMaxItems = 64;
constexpr uint32_t kPackBallotItem = 1u << 31;
constexpr uint32_t kPackLongDirection = 8;
constexpr uint32_t kSlotBatch = 4;  // link slots per pass in the slot split (Sierpinski: 32 slots, 8 warps)
constexpr uint32_t kPackStaticItems = 2;  // TileParams::pflags: compacted gathers with the static item split (A/B)
constexpr uint32_t kPackCompact = 4;      // TileParams::pflags: compacted gathers for any link-item context

// Links whose out-of-chunk gathers go to a [tile][link] (or [slot][32]) buffer; 0 = compacted buffer.
__host__ __device__ inline uint32_t pack_prefetch_links(const TileParams& p) {
  return (p.pflags & kPackCompact) ? 0u : prefetch_links(p);
}

__host__ __device__ inline uint32_t pack_zw(const TileParams& p) { return (p.Kw + p.E + 1) * 4; }

struct PackSmem {
  uint32_t* Z0;   // pstages x zw u32 (state/link/zero words)
  uint32_t zw;
  uint32_t* A0;   // kAdjSlots x ndirs x 128 adjacency words
  uint32_t* R;    // prefetched words holding out-of-chunk neighbour bits (next chunk): [4E][32]
                  // (slots), [128 tiles][E] (link items), or compacted (p.rcap words, below)
  uint32_t* rctr; // compacted R: [2] words allocated per chunk parity
  uint32_t* rb;   // compacted R: [2][kPackMaxItems] first word of each group item's gathers
  uint32_t* rbb;  // compacted R: [2][4E] first word of each (short link, lane group)'s gathers
  uint32_t* sl;   // [4E] link slot u = 4e + q: j2 << 10 | (direction * 128 + 32 q)
  uint64_t* bar;  // [pstages] state copies landed, then [kAdjSlots] adjacency copies landed
  uint32_t* items;   // [kPackMaxItems] link work items (BYDIR, see pack_link_items), then the count
  uint32_t* slinks;  // [E] the links of the short directions (ballot items)
  uint32_t ndirs, ns;
  __device__ __forceinline__ uint32_t* Z(uint32_t s) const { return Z0 + s * zw; }
  __device__ __forceinline__ const uint32_t* ntl(uint32_t a) const { return A0 + a * ndirs * kPackTiles; }
  __device__ __forceinline__ uint64_t* abar(uint32_t a) const { return bar + ns + a; }
};

__host__ __device__ inline size_t packed_layout(const TileParams& p, uint8_t* base, PackSmem* s) {
  const size_t zw = pack_zw(p);
  const size_t ns = p.pstages ? p.pstages : 2;
  size_t off = 0;
  if (s) {
    s->Z0 = (uint32_t*)base;
    s->zw = (uint32_t)zw;
    s->ndirs = p.ndirs;
    s->ns = (uint32_t)ns;
  }
  off += ns * zw * 4;
  if (s) s->A0 = (uint32_t*)(base + off);
  off += (size_t)kAdjSlots * p.ndirs * kPackTiles * 4;
  if (s) s->R = (uint32_t*)(base + off);
  off += pack_prefetch_links(p) ? (size_t)4 * pack_prefetch_links(p) * 32 * 4 : align16((size_t)(p.rcap ? p.rcap : 1) * 4);
  if (s) s->rctr = (uint32_t*)(base + off);
  off += 16;
  if (s) s->rb = (uint32_t*)(base + off);
  off += pack_prefetch_links(p) ? 0 : (size_t)2 * kPackMaxItems * 4;
  if (s) s->rbb = (uint32_t*)(base + off);
  off += pack_prefetch_links(p) ? 0 : align16((size_t)2 * 4 * (p.E ? p.E : 1) * 4);
  if (s) s->sl = (uint32_t*)(base + off);
  off += align16((size_t)(p.E ? 4 * p.E : 1) * 4);
  if (s) s->bar = (uint64_t*)(base + off);
  off += (ns + kAdjSlots) * 8;
  if (s) s->items = (uint32_t*)(base + off);
  off += (kPackMaxItems + 4) * 4;
  if (s) s->slinks = (uint32_t*)(base + off);
  off += align16((size_t)(p.E ? p.E : 1) * 4);
  return align16(off);
}

size_t packed_smem_bytes(const TileParams& p) { return packed_layout(p, nullptr, nullptr); }
bool packed_compact_gathers(const TileParams& p) { return pack_prefetch_links(p) == 0; }

// Host check of the link work items pack_link_items builds (BYDIR variants, E >= 3 ndirs): at most
// kPackMaxItems of them, link indices below 2^11 (their 11-bit fields).  Contexts that fail it (a
// line-like fractal whose tile is nearly all boundary) leave the packed step unavailable.
bool packed_items_fit(const uint16_t* dir_start, uint32_t ndirs, uint32_t E, uint32_t nwarps) {
  if (E < 3 * ndirs) return true;  // slot split: no items
  if (E >= 2048 || nwarps == 0) return false;
  uint32_t n = 0, ns = 0;
  for (uint32_t d = 0; d < ndirs; ++d) {
    const uint32_t nd = (uint32_t)dir_start[d + 1] - dir_start[d];
    if (nd == 0) continue;
    if (nd < kPackLongDirection) ns += nd;
    else n += 4 * ((nd + 31) / 32);
  }
  const uint32_t free_w = nwarps - n % nwarps;
  return n + (ns == 0 ? 0u : std::min(ns, free_w)) <= kPackMaxItems;
}

__host__ __device__ inline uint64_t pack_chunks(const TileParams& p) {
  return (p.tile_hi - p.tile_lo + kPackTiles - 1) / kPackTiles;
}

struct PackChunk {
  uint64_t c;
  uint32_t t0;  // first tile (tile indices < 2^32, checked on the host)
  uint32_t nt;  // tiles in the chunk
};

__device__ __forceinline__ PackChunk pack_chunk(const TileParams& p, uint64_t c) {
  PackChunk pc;
  pc.c = c;
  const uint64_t t0 = p.tile_lo + c * kPackTiles;
  pc.t0 = (uint32_t)t0;
  pc.nt = (uint32_t)min((uint64_t)kPackTiles, p.tile_hi - t0);
  return pc;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One thread: the chunk's Kw words -> state stage s.
__device__ __forceinline__ void state_load(const TileParams& p, const PackSmem& S, const PackChunk& pc, uint32_t s,
                                           const uint4* __restrict__ cur) {
  const uint32_t bytes = p.Kw * 16;
  uint64_t* bar = &S.bar[s];
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  bulk_g2s(smem_u32(S.Z(s)), cur + pc.c * p.Kw, bytes, bar);
}

// One thread: the chunk's 128 adjacency words per link direction -> adjacency slot a.
// (Adjacency rows are padded to whole chunks on the host, so every copy is 512 bytes.)
__device__ __forceinline__ void adj_load(const TileParams& p, const PackSmem& S, const PackChunk& pc, uint32_t a) {
  const uint32_t abytes = kPackTiles * 4;
  uint64_t* bar = S.abar(a);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(abytes * p.ndirs)
               : "memory");
  const uint32_t dst = smem_u32(S.ntl(a));
  for (uint32_t d = 0; d < p.ndirs; ++d)
    bulk_g2s(dst + d * abytes, p.adj + d * p.adj_stride + (pc.t0 - p.tile_lo), abytes, bar);
}

// Link slot u = 4e + q: link e for the 32 tiles of lane group q (tiles 32q..32q+31 of the chunk).
// Two work splits.  SLOTS: slot u belongs to warp u mod W (few links per direction, e.g. the
// Sierpinski triangle's 8 links).  BYDIR: link work items (below; link-heavy fractals such as the
// carpet's 112 links per tile).  Either way a slot/item belongs to the same warp here and in the
// link phase of the next iteration (same thread: program order suffices).  For a link whose neighbour tile is outside the chunk: a 4-byte
// cp.async of the packed word holding the neighbour bit.  `ntl` = the chunk's adjacency words
// (neighbour tile + 1, from the coarse λ + ν at init: P:189 at tile level).  Commits one group.
template <bool SHARDED>
__device__ __forceinline__ void chunk_prefetch_slots(const TileParams& p, const PackSmem& S, const PackChunk& pc,
                                               const uint32_t* ntl, const uint32_t* __restrict__ cur32, int warp,
                                               int nwarps, int lane) {
  const uint32_t E = pack_prefetch_links(p);
#pragma unroll 4
  for (uint32_t u = (uint32_t)warp; u < 4 * E; u += (uint32_t)nwarps) {
    const uint32_t sl = S.sl[u];
    const uint32_t a1 = ntl[(sl & 1023u) + lane];
    const uint32_t tl = a1 - 1u - (uint32_t)p.tile_lo;
    if (a1 != 0 && a1 - 1u - pc.t0 >= pc.nt) {
      if (!SHARDED || tl < (uint32_t)(p.tile_hi - p.tile_lo))
        cp_async4(&S.R[u * 32 + lane], cur32 + ((uint64_t)(tl >> 7) * p.Kw + (sl >> 10)) * 4 + ((tl >> 5) & 3u));
      else  // another shard's tile (sharded contexts): the bit from the halo, placed where the link reads it
        S.R[u * 32 + lane] = halo_fetch(p.halo, (uint64_t)(a1 - 1u) * p.K + (sl >> 10)) << (tl & 31u);
    }
  }
  cp_async_commit();
}

// BYDIR link work items (link-heavy fractals).  A GROUP item (bit 31 clear: first
// link | count - 1 << 11 | direction << 16 | lane group q << 24) holds up to 32 links of one long
// direction for the 32 tiles of lane group q (four items per link group: finer work units balance
// the warps in front of the chunk barrier); lane = link.
// A direction's neighbour tiles are the same for all its links, so per (group, lane group q, tile)
// the work is warp-uniform: the in-chunk part of a link word is a few masked rotations of the
// neighbour cell's state word (one per distinct (source lane group, offset) of the tiles of q),
// the out-of-chunk part one gathered word per outside tile.  A BALLOT item (bit 31 set: first index
// into slinks | count - 1 << 11) holds links of the short directions (a corner's single link),
// lane = tile, one ballot per (link, q).  R holds the gathers as [tile t of the chunk][link e], or
// compacted (chunk_prefetch_items).
__device__ void pack_link_items(const TileParams& p, const PackSmem& S, uint32_t nwarps) {  // one thread
  uint32_t n = 0, ns = 0;
  for (uint32_t d = 0; d < p.ndirs; ++d) {
    const uint32_t e0 = p.dir_start[d], e1 = p.dir_start[d + 1], nd = e1 - e0;
    if (nd == 0) continue;
    if (nd < kPackLongDirection) {
      for (uint32_t e = e0; e < e1; ++e) S.slinks[ns++] = e;
      continue;
    }
    const uint32_t ng = (nd + 31) / 32;  // groups of balanced sizes
    for (uint32_t k = 0, e = e0; k < ng; ++k) {
      const uint32_t m = (nd - (e - e0) + (ng - k) - 1) / (ng - k);
      for (uint32_t q = 0; q < 4; ++q) S.items[n++] = e | ((m - 1u) << 11) | (d << 16) | (q << 24);
      e += m;
    }
  }
  const uint32_t free_w = nwarps - n % nwarps;  // short links: ballot items on the warps of the last round
  const uint32_t nb = ns == 0 ? 0u : min(ns, free_w);
  for (uint32_t k = 0, i = 0; k < nb; ++k) {
    const uint32_t m = (ns - i + (nb - k) - 1) / (nb - k);
    S.items[n++] = kPackBallotItem | i | ((m - 1u) << 11);
    i += m;
  }
  S.items[kPackMaxItems] = n;
}

// The packed word holding the neighbour bit (tile tl of the shard, cell j2), read synchronously: a
// compacted gather buffer's overflow.  Another shard's tile (sharded contexts): the bit from the
// halo, placed where the link reads it (bit tl mod 32).
template <bool SHARDED>
__device__ __forceinline__ uint32_t link_gather(const TileParams& p, const uint32_t* __restrict__ cur32, uint32_t tl,
                                                uint32_t j2, uint32_t nloc) {
  if (SHARDED && tl >= nloc) return halo_fetch(p.halo, (uint64_t)(tl + (uint32_t)p.tile_lo) * p.K + j2) << (tl & 31u);
  return __ldg(cur32 + ((uint64_t)(tl >> 7) * p.Kw + j2) * 4 + ((tl >> 5) & 3u));
}

// Gathers of chunk pc's out-of-chunk links (issued one chunk ahead).  With E <= kMaxPrefetchLinks
// R is [tile t of the chunk][link e].  Above that (the carpet at level 4: 328 links, a [128][E]
// buffer would be 168 KB) R is COMPACTED: only the (outside tile, link) pairs the chunk has get a
// word.  Each item takes its words with one shared atomicAdd on the chunk parity's counter and
// records where they start (rb / rbb); the words of its r-th outside tile (in ballot order) are
// base + r n + link.  Pairs past p.rcap are not prefetched: the link item reads them synchronously
// (link_gather).  Producer and consumer of a word are the same lane (same item-to-warp split).
template <bool SHARDED>
__device__ __forceinline__ void chunk_prefetch_items(const TileParams& p, const PackSmem& S, const PackChunk& pc,
                                                     const uint32_t* ntl, const uint32_t* __restrict__ cur32,
                                                     int warp, int nwarps, int lane, uint32_t par, uint32_t ro,
                                                     uint32_t rcap) {
  // compacted: words [ro, ro + rcap) of R (ro = 0, rcap = p.rcap; or one parity's half, DYN)
  const uint32_t E = p.E, ni = S.items[kPackMaxItems], tlo = (uint32_t)p.tile_lo, Kw = p.Kw;
  const uint32_t nloc = (uint32_t)(p.tile_hi - p.tile_lo), gs0 = smem_u32(S.R);
  const bool compact = pack_prefetch_links(p) == 0;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t k = (uint32_t)warp; k < ni; k += (uint32_t)nwarps) {
    const uint32_t item = S.items[k], i0 = item & 0x7FFu, n = ((item >> 11) & 31u) + 1u;
    if (item & kPackBallotItem) {  // lane = tile, link by link
      for (uint32_t i = i0; i < i0 + n; ++i) {
        const uint32_t e = S.slinks[i], sl = S.sl[4 * e], d = (sl & 1023u) >> 7, j2 = sl >> 10;  // (lane group 0's slot)
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          const uint32_t a1 = ntl[d * kPackTiles + q * 32 + lane], tl = a1 - 1u - tlo, t = q * 32 + lane;
          const bool out = a1 != 0 && a1 - 1u - pc.t0 >= pc.nt;
          uint32_t slot = t * E + e;
          bool fits = true;
          if (compact) {
            const uint32_t om = __ballot_sync(0xFFFFFFFFu, out);
            uint32_t base = 0;
            if (lane == 0 && om) base = atomicAdd(&S.rctr[par], (uint32_t)__popc(om));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (lane == 0) S.rbb[par * 4 * E + i * 4 + q] = base;
            slot = base + (uint32_t)__popc(om & lt);
            fits = slot < rcap;
            slot += ro;
          }
          if (SHARDED && out && fits && tl >= nloc) S.R[slot] = halo_fetch(p.halo, (uint64_t)(a1 - 1u) * p.K + j2) << (tl & 31u);
          else cp_async4_if(gs0 + 4u * (fits ? slot : 0u), cur32 + ((uint64_t)((out ? tl : 0u) >> 7) * Kw + j2) * 4 + ((tl >> 5) & 3u),
                            out && fits ? 1u : 0u);
        }
      }
      continue;
    }
    const uint32_t d = (item >> 16) & 0xFFu, q = (item >> 24) & 3u, valid = (uint32_t)lane < n ? 1u : 0u;
    const uint32_t e = i0 + (valid ? (uint32_t)lane : 0u), j2 = S.sl[4 * e] >> 10;
    {
      const uint32_t a1 = ntl[d * kPackTiles + q * 32 + lane], tl = a1 - 1u - tlo;  // lane = tile here
      const bool out = a1 != 0 && a1 - 1u - pc.t0 >= pc.nt;
      uint32_t om = __ballot_sync(0xFFFFFFFFu, out);
      const uint32_t farm = SHARDED ? __ballot_sync(0xFFFFFFFFu, out && tl >= nloc) : 0u;
      uint32_t br = 0;  // compacted: first word of the current outside tile's n links
      if (compact) {
        const uint32_t cnt = (uint32_t)__popc(om) * n;
        if (lane == 0 && cnt) br = atomicAdd(&S.rctr[par], cnt);
        br = __shfl_sync(0xFFFFFFFFu, br, 0);
        if (lane == 0) S.rb[par * kPackMaxItems + k] = br;
      }
      // the source word of tile tli: this link's word of chunk tli / 128, u32 lane (tli / 32) mod 4
      const uint64_t gb = reinterpret_cast<uint64_t>(cur32) + (uint64_t)j2 * 16u;
      const uint32_t kw16 = Kw * 16u;
      while (om) {  // lane = link from here on
        const uint32_t i = __ffs(om) - 1u;
        om &= om - 1u;
        const uint32_t tli = __shfl_sync(0xFFFFFFFFu, tl, i), t = q * 32 + i;
        const uint32_t slot = compact ? ro + br + (uint32_t)lane : t * E + e;
        const uint32_t ok = compact ? (br + n <= rcap ? valid : 0u) : valid;
        br += n;
        if (!SHARDED || !((farm >> i) & 1u))
          cp_async4_if(gs0 + 4u * (ok ? slot : 0u),
                       reinterpret_cast<const void*>(gb + (uint64_t)(tli >> 7) * kw16 + ((tli >> 3) & 12u)), ok);
        else if (ok)  // another shard's tile (sharded contexts): the bit from the halo, placed where it is read
          S.R[slot] = halo_fetch(p.halo, (uint64_t)(tli + tlo) * p.K + j2) << (tli & 31u);
      }
    }
  }
  cp_async_commit();
}

// Link words of chunk pc (BYDIR items): bit i of u32 lane q of word Kw + e = cell j2 of the
// neighbour tile (link e) of tile 32q + i.
template <bool SHARDED>
// dctr != nullptr (DYN): items are taken dynamically from that shared counter (their gathers were
// completed before a CTA barrier, so any warp may read them); else item k belongs to warp k mod W.
__device__ __forceinline__ void chunk_link_items(const TileParams& p, const PackSmem& S, const PackChunk& pc,
                                                 const uint32_t* ntl, uint32_t* Z, const uint32_t* __restrict__ cur32,
                                                 int warp, int nwarps, int lane, uint32_t par, uint32_t ro,
                                                 uint32_t rcap, uint32_t* dctr) {
  const uint32_t E = p.E, ni = S.items[kPackMaxItems], tlo = (uint32_t)p.tile_lo, Kw = p.Kw;
  const bool compact = pack_prefetch_links(p) == 0;
  const uint32_t lt = (1u << lane) - 1u, nloc = (uint32_t)(p.tile_hi - p.tile_lo);
  auto grab = [&]() -> uint32_t {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(dctr, 1u);
    return __shfl_sync(0xFFFFFFFFu, v, 0);
  };
  for (uint32_t k = dctr ? grab() : (uint32_t)warp; k < ni; k = dctr ? grab() : k + (uint32_t)nwarps) {
    const uint32_t item = S.items[k], i0 = item & 0x7FFu, n = ((item >> 11) & 31u) + 1u;
    if (item & kPackBallotItem) {  // lane = tile, one ballot per (link, q)
      for (uint32_t i = i0; i < i0 + n; ++i) {
        const uint32_t e = S.slinks[i], sl = S.sl[4 * e], d = (sl & 1023u) >> 7, j2 = sl >> 10;  // (lane group 0's slot)
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          const uint32_t a1 = ntl[d * kPackTiles + q * 32 + lane], rel = a1 - 1u - pc.t0, tl = a1 - 1u - tlo;
          const bool in = rel < pc.nt;
          uint32_t g;
          if (compact) {
            const uint32_t om = __ballot_sync(0xFFFFFFFFu, a1 != 0 && !in);
            const uint32_t slot = S.rbb[par * 4 * E + i * 4 + q] + (uint32_t)__popc(om & lt);
            g = a1 == 0 || in ? 0u : slot < rcap ? S.R[ro + slot] : link_gather<SHARDED>(p, cur32, tl, j2, nloc);
          } else {
            g = a1 == 0 || in ? 0u : S.R[(q * 32 + lane) * E + e];
          }
          const uint32_t v = a1 == 0 ? 0u : in ? Z[j2 * 4 + (rel >> 5)] >> (rel & 31u) : g >> (tl & 31u);
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v & 1u);
          if (lane == 0) Z[(Kw + e) * 4 + q] = bal;
        }
      }
      continue;
    }
    const uint32_t d = (item >> 16) & 0xFFu, q = (item >> 24) & 3u, valid = (uint32_t)lane < n ? 1u : 0u;
    const uint32_t e = i0 + (valid ? (uint32_t)lane : 0u), j2 = S.sl[4 * e] >> 10;
    const uint4 z = *reinterpret_cast<const uint4*>(Z + j2 * 4);  // the neighbour cell's word, all 128 tiles
    {
      const uint32_t a1 = ntl[d * kPackTiles + q * 32 + lane], rel = a1 - 1u - pc.t0, tl = a1 - 1u - tlo;  // lane = tile
      const bool present = a1 != 0, inside = present && rel < pc.nt;
      const uint32_t key = (rel & ~31u) | ((rel - (uint32_t)lane) & 31u);  // source lane group, offset
      uint32_t im = __ballot_sync(0xFFFFFFFFu, inside);
      uint32_t om = __ballot_sync(0xFFFFFFFFu, present && !inside);
      uint32_t w = 0;
      while (im) {  // tiles with the same (source group, offset): one masked rotation
        const uint32_t kk = __shfl_sync(0xFFFFFFFFu, key, __ffs(im) - 1u);
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, inside && key == kk);
        im &= ~m;
        const uint32_t lo = (kk & 32u) ? z.y : z.x, hi = (kk & 32u) ? z.w : z.z;  // source group kk >> 5, by selects
        const uint32_t src = (kk & 64u) ? hi : lo;
        w |= __funnelshift_r(src, src, kk & 31u) & m;
      }
      if (compact) {  // the gathered words of the outside tiles, in the prefetch's order
        uint32_t br = S.rb[par * kPackMaxItems + k];
        while (om) {  // two outside tiles at a time (independent loads)
          const uint32_t i = __ffs(om) - 1u;
          om &= om - 1u;
          const bool two = om != 0u;
          const uint32_t i2 = two ? __ffs(om) - 1u : i;
          om &= om - 1u;
          const uint32_t t1 = __shfl_sync(0xFFFFFFFFu, tl, i), t2 = __shfl_sync(0xFFFFFFFFu, tl, i2);
          const uint32_t b1 = br, b2 = two ? br + n : br;
          br = b2 + n;
          const uint32_t g1 = !valid ? 0u : b1 + n <= rcap ? S.R[ro + b1 + lane] : link_gather<SHARDED>(p, cur32, t1, j2, nloc);
          const uint32_t g2 = !valid ? 0u : b2 + n <= rcap ? S.R[ro + b2 + lane] : link_gather<SHARDED>(p, cur32, t2, j2, nloc);
          w |= (((g1 >> (t1 & 31u)) & 1u) << i) | (((g2 >> (t2 & 31u)) & 1u) << i2);
        }
      }
      while (om) {  // tiles whose neighbour tile is outside the chunk: the gathered words, two at a time
        const uint32_t i = __ffs(om) - 1u;
        om &= om - 1u;
        const uint32_t i2 = om ? __ffs(om) - 1u : i;
        om &= om - 1u;
        const uint32_t sh = __shfl_sync(0xFFFFFFFFu, tl, i) & 31u, sh2 = __shfl_sync(0xFFFFFFFFu, tl, i2) & 31u;
        const uint32_t g1 = valid ? S.R[(q * 32 + i) * E + e] : 0u, g2 = valid ? S.R[(q * 32 + i2) * E + e] : 0u;
        w |= (((g1 >> sh) & 1u) << i) | (((g2 >> sh2) & 1u) << i2);
      }
      if (valid) Z[(Kw + e) * 4 + q] = w;
    }
  }
}

template <bool SHARDED, bool BYDIR>
__device__ __forceinline__ void chunk_prefetch(const TileParams& p, const PackSmem& S, const PackChunk& pc,
                                               const uint32_t* ntl, const uint32_t* __restrict__ cur32, int warp,
                                               int nwarps, int lane, uint32_t par, uint32_t ro, uint32_t rcap) {
  if (BYDIR) chunk_prefetch_items<SHARDED>(p, S, pc, ntl, cur32, warp, nwarps, lane, par, ro, rcap);
  else chunk_prefetch_slots<SHARDED>(p, S, pc, ntl, cur32, warp, nwarps, lane);
}

// Carry-save count of DMAX neighbour words and the rule, on one 32-bit lane of the word.
template <int DMAX, bool CONWAY>
__device__ __forceinline__ uint32_t cell_rule(const uint32_t* x, uint32_t alive, uint32_t birth, uint32_t survive) {
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
  if (CONWAY) return c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23: count 3, or count 2 and alive
  return (alive & rule_bits(survive, c0, c1, c2, c3)) | (~alive & rule_bits(birth, c0, c1, c2, c3));
}

// ------------------------------------------------------------------------------------ step
// DMAX: neighbour slots per cell (5 for the Sierpinski triangle, else 8).  RB: j-blocks per warp
// whose neighbour slots stay in registers for the whole launch (block jb = warp + i * W); later
// blocks read their slots through L1.
// DYN (link items with compacted gathers, one CTA per SM): the out-of-chunk gathers run TWO chunks
// ahead into R halves by chunk parity and complete before the chunk barrier in between, so the link
// items of a chunk can be taken dynamically by whichever warp is free (the static split left 21% of
// the carpet's stall samples at the chunk barrier, waiting for the warps with the costliest items).
template <int DMAX, bool CONWAY, int RB, int MAXT, int MINB, bool SHARDED, bool BYDIR, bool DYN>
__global__ void __launch_bounds__(MAXT, MINB) k_step_packed(TileParams p, const uint4* __restrict__ cur,
                                                        uint4* __restrict__ next) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PackSmem S;
  packed_layout(p, smem_raw, &S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K, Kw = p.Kw, E = p.E, NS = p.pstages;
  const uint32_t Epf = pack_prefetch_links(p);
  const uint64_t nch = pack_chunks(p);
  const bool issuer = warp == nwarps - 1 && lane == 0;
  const uint32_t* cur32 = reinterpret_cast<const uint32_t*>(cur);
  const uint32_t nloc = (uint32_t)(p.tile_hi - p.tile_lo);  // local tiles

  uint32_t off[RB][DMAX];  // byte offsets of this lane's neighbour words in a stage (slot x 16)
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const uint32_t j = ((uint32_t)warp + (uint32_t)(i * nwarps)) * 32 + lane;
    const uint4 row = j < K ? __ldg(reinterpret_cast<const uint4*>(p.nbr) + j) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {row.x, row.y, row.z, row.w};
#pragma unroll
    for (int k = 0; k < DMAX; ++k) off[i][k] = ((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) * 16;
  }

  uint32_t fullmask = 0;  // blocks i < RB whose 32 words are all cells
#pragma unroll
  for (int i = 0; i < RB; ++i)
    if (((uint32_t)warp + (uint32_t)(i * nwarps) + 1) * 32 <= K) fullmask |= 1u << i;
  for (uint32_t i = tid; i < NS * 4; i += blockDim.x) S.Z(i >> 2)[(Kw + E) * 4 + (i & 3)] = 0;  // zero slot
  for (uint32_t u = tid; u < 4 * E; u += blockDim.x)
    S.sl[u] = (p.link_j2[u >> 2] << 10) | (p.link_dir[u >> 2] * kPackTiles + 32 * (u & 3u));
  if (tid == 0) {
    S.rctr[0] = S.rctr[1] = S.rctr[2] = S.rctr[3] = 0;  // allocation counters, DYN item counters
    if (BYDIR) pack_link_items(p, S, (uint32_t)nwarps);
    for (uint32_t s = 0; s < NS + kAdjSlots; ++s) mbar_init(&S.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t c = blockIdx.x;
  if (c >= nch) return;
  const uint64_t G = gridDim.x;
  if (issuer) {
    for (uint32_t s = 0; s + 1 < NS && c + s * G < nch; ++s) state_load(p, S, pack_chunk(p, c + s * G), s, cur);
    for (uint32_t a = 0; a + 1 < kAdjSlots && c + a * G < nch; ++a) adj_load(p, S, pack_chunk(p, c + a * G), a);
  }
  const uint32_t rh = DYN ? (p.rcap / 2) & ~31u : p.rcap;  // DYN: R in two halves by chunk parity
  auto ro_of = [&](uint32_t par) -> uint32_t { return DYN ? par * rh : 0u; };
  mbar_wait(S.abar(0), 0);
  chunk_prefetch<SHARDED, BYDIR>(p, S, pack_chunk(p, c), S.ntl(0), cur32, warp, nwarps, lane, 0u, 0u, rh);
  if (DYN) {  // the second chunk's gathers too; both complete before the first chunk's link items
    if (c + G < nch) {
      mbar_wait(S.abar(1), 0);
      chunk_prefetch<SHARDED, BYDIR>(p, S, pack_chunk(p, c + G), S.ntl(1), cur32, warp, nwarps, lane, 1u, ro_of(1), rh);
    }
    cp_async_wait_all();
    __syncthreads();
  }

  uint32_t it = 0, s = 0, sphase = 0;  // sphase bit s: parity of state stage s's next completion
  for (; c < nch; c += G, ++it, s = (s + 1 == NS) ? 0 : s + 1) {
    const PackChunk pc = pack_chunk(p, c);
    uint32_t* Z = S.Z(s);
    const uint32_t zs = __reduce_or_sync(0xFFFFFFFFu, smem_u32(Z));  // warp-uniform: a uniform register, folded into the LDS addresses
    const uint32_t a = it & (kAdjSlots - 1);
    const uint32_t* ntl = S.ntl(a);
    mbar_wait(&S.bar[s], (sphase >> s) & 1);
    sphase ^= 1u << s;

    // link words: bit i of u32 lane q of word Kw + e = cell j2 of the neighbour tile (link e)
    // of tile 32q + i
    // compacted R: the counter chunk it+1's (DYN: it+2's) prefetch allocates from
    if (tid == 0) S.rctr[DYN ? (it & 1u) : ((it + 1) & 1u)] = 0;
    if (BYDIR) {
      if (DYN || (uint32_t)warp < S.items[kPackMaxItems]) {
        mbar_wait(S.abar(a), (it / kAdjSlots) & 1);  // (already complete when the prefetch ran)
        if (!DYN) cp_async_wait_all();
        chunk_link_items<SHARDED>(p, S, pc, ntl, Z, cur32, warp, nwarps, lane, it & 1u, ro_of(it & 1u), rh,
                                  DYN ? &S.rctr[2 + (it & 1u)] : nullptr);
      }
    } else {
    if ((uint32_t)warp < 4 * E) {
      mbar_wait(S.abar(a), (it / kAdjSlots) & 1);  // (already complete when the prefetch ran)
      cp_async_wait_all();
      const uint32_t rs = smem_u32(S.R) + lane * 4;
      const uint32_t ntl_s = smem_u32(ntl) + lane * 4;
      // kSlotBatch slots per pass, their loads issued together (independent chains: the link phase
      // sits in front of the chunk barrier, so its latency, not its instruction count, matters).
      // The slot split only runs with every link prefetched (E < 3 ndirs <= 24 <= kMaxPrefetchLinks).
      const uint32_t zl = zs + 16u * Kw, m1t0 = ~pc.t0, m1tlo = ~(uint32_t)p.tile_lo, nt = pc.nt;
      for (uint32_t u0 = (uint32_t)warp; u0 < 4 * E; u0 += kSlotBatch * (uint32_t)nwarps) {
        uint32_t v[kSlotBatch];
#pragma unroll
        for (uint32_t k = 0; k < kSlotBatch; ++k) {
          const uint32_t u0k = u0 + k * (uint32_t)nwarps, u = u0k < 4 * E ? u0k : 0u;  // branch-free: straight-line
          const uint32_t sl = S.sl[u];                                                   // code interleaves the slots' loads
          const uint32_t a1 = lds32(ntl_s + (sl & 1023u) * 4);
          const uint32_t rel = a1 + m1t0;  // neighbour tile - t0 (a1 = tile + 1)
          const bool in = rel < nt;
          const uint32_t w = lds32(in ? zs + (sl >> 10) * 16 + ((rel >> 3) & ~3u) : rs + u * 128);
          const uint32_t sh = in ? rel : a1 + m1tlo;
          v[k] = a1 != 0 && u0k < 4 * E ? (w >> (sh & 31u)) & 1u : 0u;
        }
#pragma unroll
        for (uint32_t k = 0; k < kSlotBatch; ++k) {
          const uint32_t u = u0 + k * (uint32_t)nwarps;
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v[k] != 0);
          if (lane == 0 && u < 4 * E) sts32(zl + 4 * u, bal);
        }
      }
    }
    }
    if (DYN) cp_async_wait_all();  // this warp's gathers of chunk it+1 (issued an iteration ago)
    __syncthreads();  // the one CTA barrier per chunk: state + link words in place, chunk it-1 done
    if (DYN && tid == 0) S.rctr[2 + (it & 1u)] = 0;  // the item counter, for chunk it+2
    if (issuer) {
      if (c + (NS - 1) * G < nch) {
        fence_proxy_async();
        state_load(p, S, pack_chunk(p, c + (NS - 1) * G), (s + NS - 1) % NS, cur);
      }
      if (c + (kAdjSlots - 1) * G < nch)
        adj_load(p, S, pack_chunk(p, c + (kAdjSlots - 1) * G), (it + kAdjSlots - 1) & (kAdjSlots - 1));
    }
    // out-of-chunk link gathers of the next chunk (DYN: the one after; its adjacency was issued long ago)
    if (c + (DYN ? 2 : 1) * G < nch) {
      const uint32_t itn = it + (DYN ? 2u : 1u), a1 = itn & (kAdjSlots - 1);
      if (DYN || (BYDIR ? (uint32_t)warp < S.items[kPackMaxItems] : ((uint32_t)warp < 4 * Epf && Epf)))
        mbar_wait(S.abar(a1), (itn / kAdjSlots) & 1);
      chunk_prefetch<SHARDED, BYDIR>(p, S, pack_chunk(p, c + (DYN ? 2 : 1) * G), S.ntl(a1), cur32, warp, nwarps,
                                     lane, itn & 1u, ro_of(itn & 1u), rh);
    }

    // count + rule: lane = word j (128 cells), straight to HBM
    uint4 lm = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (pc.nt < kPackTiles) {  // the shard's last chunk: bits of tiles past its end stay 0
      const uint32_t n = pc.nt;
      lm.x = n >= 32 ? ~0u : (1u << n) - 1u;
      lm.y = n >= 64 ? ~0u : (n <= 32 ? 0u : (1u << (n - 32)) - 1u);
      lm.z = n >= 96 ? ~0u : (n <= 64 ? 0u : (1u << (n - 64)) - 1u);
      lm.w = n <= 96 ? 0u : (1u << (n - 96)) - 1u;
    }
    uint4* outc = next + pc.c * Kw;
    auto word = [&](uint32_t j, const uint32_t* o) {
      if (j >= Kw) return;
      uint4 nw = make_uint4(0, 0, 0, 0);
      if (j < K) {
        uint32_t x0[DMAX], x1[DMAX], x2[DMAX], x3[DMAX];
#pragma unroll
        for (int k = 0; k < DMAX; ++k) {
          const uint4 v = lds128(zs + o[k]);
          x0[k] = v.x;
          x1[k] = v.y;
          x2[k] = v.z;
          x3[k] = v.w;
        }
        const uint4 al = lds128(zs + j * 16);
        nw.x = cell_rule<DMAX, CONWAY>(x0, al.x, p.birth, p.survive);
        nw.y = cell_rule<DMAX, CONWAY>(x1, al.y, p.birth, p.survive);
        nw.z = cell_rule<DMAX, CONWAY>(x2, al.z, p.birth, p.survive);
        nw.w = cell_rule<DMAX, CONWAY>(x3, al.w, p.birth, p.survive);
        // the shard's last chunk: bits of tiles past its end stay 0.  Under B3/S23 they do so anyway
        // (their state bits and link bits are 0, so their count is 0: no birth)
        if (!CONWAY && pc.nt < kPackTiles) {
          nw.x &= lm.x;
          nw.y &= lm.y;
          nw.z &= lm.z;
          nw.w &= lm.w;
        }
      }
      outc[j] = nw;  // padding words K..Kw-1 are written 0
    };
    auto word_full = [&](uint32_t j, const uint32_t* o) {  // a block whose 32 words are all cells (j < K)
      uint32_t x0[DMAX], x1[DMAX], x2[DMAX], x3[DMAX];
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        const uint4 v = lds128(zs + o[k]);
        x0[k] = v.x;
        x1[k] = v.y;
        x2[k] = v.z;
        x3[k] = v.w;
      }
      const uint4 al = lds128(zs + j * 16);
      uint4 nw;
      nw.x = cell_rule<DMAX, CONWAY>(x0, al.x, p.birth, p.survive);
      nw.y = cell_rule<DMAX, CONWAY>(x1, al.y, p.birth, p.survive);
      nw.z = cell_rule<DMAX, CONWAY>(x2, al.z, p.birth, p.survive);
      nw.w = cell_rule<DMAX, CONWAY>(x3, al.w, p.birth, p.survive);
      if (!CONWAY && pc.nt < kPackTiles) {
        nw.x &= lm.x;
        nw.y &= lm.y;
        nw.z &= lm.z;
        nw.w &= lm.w;
      }
      outc[j] = nw;
    };
    // blocks past the register-resident ones read their neighbour-table rows through L1, one block
    // ahead (the first one issued before the register blocks), so the load latency is hidden
    // (large-tile variants only: the small-tile ones, three CTAs per SM, hold every block's slots in
    // registers, and the extra live row cost them 3% at the carpet's level 3)
    constexpr bool kRowAhead = MINB < 3;
    const uint4* nbr4 = reinterpret_cast<const uint4*>(p.nbr);
    uint32_t jb = (uint32_t)warp + (uint32_t)(RB * nwarps);
    uint4 rown = make_uint4(0, 0, 0, 0);
    if (kRowAhead && jb * 32 + lane < K) rown = __ldg(nbr4 + jb * 32 + lane);
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const uint32_t j = ((uint32_t)warp + (uint32_t)(i * nwarps)) * 32 + lane;
      if ((fullmask >> i) & 1u) word_full(j, off[i]);
      else word(j, off[i]);
    }
    for (; jb * 32 < Kw; jb += (uint32_t)nwarps) {
      const uint32_t j = jb * 32 + lane, jn = j + 32 * (uint32_t)nwarps;
      uint4 row;
      if (kRowAhead) {
        row = rown;
        rown = jn < K ? __ldg(nbr4 + jn) : make_uint4(0, 0, 0, 0);
      } else {
        row = j < K ? __ldg(nbr4 + j) : make_uint4(0, 0, 0, 0);
      }
      const uint32_t w[4] = {row.x, row.y, row.z, row.w};
      uint32_t o[DMAX];
#pragma unroll
      for (int k = 0; k < DMAX; ++k) o[k] = ((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) * 16;
      word(j, o);
    }
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------------------------ conversions
// The conversions walk 32-tile slices: slice v = 4c + q of the shard is u32 lane q of chunk c,
// so u32 word j of slice v sits at index (c * Kw + j) * 4 + q of the packed buffer.
__device__ __forceinline__ uint64_t slice_word(const TileParams& p, uint64_t v, uint32_t j) {
  return ((v >> 2) * p.Kw + j) * 4 + (v & 3);
}

// byte layout -> packed: lane = tile reads its 32-byte window (two 128-bit loads), packs, and
// the warp transposes so lane L holds word j0 + my_jj(L).  One warp per (slice, j-block).
__global__ void k_pack(TileParams p, const uint8_t* __restrict__ st, uint32_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x >> 5;
  const uint32_t K = (uint32_t)p.K, nblk = (K + 31) / 32, wpc = (p.Kw + 31) / 32;  // blocks incl. padding words
  const uint32_t my_jj = 4 * (lane & 7) + (lane >> 3);
  const Transposer tr(lane);
  const uint64_t ntiles = p.tile_hi - p.tile_lo, nslices = pack_chunks(p) * 4;
  for (uint64_t wi = gw; wi < nslices * wpc; wi += nw) {
    const uint64_t v = wi / wpc;
    const uint32_t jb = (uint32_t)(wi - v * wpc), j0 = jb * 32;
    const uint64_t t = v * 32 + lane;
    uint32_t acc = 0;
    if (jb < nblk && t < ntiles) {
      const uint4* src = reinterpret_cast<const uint4*>(st + t * p.Kp + j0);
      const uint4 lo = __ldg(src), hi = __ldg(src + 1);
      acc = (lo.x & 0x01010101u) | ((lo.y & 0x01010101u) << 1) | ((lo.z & 0x01010101u) << 2) |
            ((lo.w & 0x01010101u) << 3) | ((hi.x & 0x01010101u) << 4) | ((hi.y & 0x01010101u) << 5) |
            ((hi.z & 0x01010101u) << 6) | ((hi.w & 0x01010101u) << 7);
    }
    const uint32_t x = tr(acc);  // bytes past K are zero in the byte layout
    if (j0 + my_jj < p.Kw) packed[slice_word(p, v, j0 + my_jj)] = x;
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
  const uint64_t ntiles = p.tile_hi - p.tile_lo, nslices = (ntiles + 31) / 32;
  const uint32_t jobs = (wpt + 1) / 2;  // 32-byte windows per tile (the last may be 16 bytes)
  for (uint64_t wi = gw; wi < nslices * jobs; wi += nw) {
    const uint64_t v = wi / jobs;
    const uint32_t jb = (uint32_t)(wi - v * jobs), j0 = jb * 32;
    uint32_t x = (jb < nblk && j0 + my_jj < K) ? packed[slice_word(p, v, j0 + my_jj)] : 0u;
    x = tr(x);
    const uint64_t t = v * 32 + lane;
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
  const uint64_t ntiles = p.tile_hi - p.tile_lo, nslices = pack_chunks(p) * 4;
  for (uint64_t wi = gw; wi < nslices * p.Kw; wi += nw) {
    const uint64_t v = wi / p.Kw;
    const uint32_t j = (uint32_t)(wi - v * p.Kw);
    const uint64_t t = v * 32 + lane;
    uint32_t a = 0;
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
      a = (h >> 32) < q ? 1u : 0u;
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, a != 0);
    if (lane == 0) packed[slice_word(p, v, j)] = bal;
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

// send[i] = state bit i of the packed state (sharded contexts: the halo this shard sends).
__global__ void k_halo_pack_packed(const uint32_t* __restrict__ cur, const uint64_t* __restrict__ bits, uint64_t n,
                                   uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = bits[i];
    out[i] = (uint8_t)((cur[b >> 5] >> (b & 31)) & 1u);
  }
}

// ------------------------------------------------------------------------------------ launchers
using PackedFn = void (*)(TileParams, const uint4*, uint4*);

// RB = j-blocks per warp with register-resident neighbour slots (ceil(nblk / W), capped).
template <bool SH, bool BD>
static PackedFn pick_packed_t(const TileParams& p, int threads) {
  const bool conway = (p.birth == (1u << 3)) && (p.survive == ((1u << 2) | (1u << 3)));
  const uint32_t nblk = (uint32_t)((p.Kw + 31) / 32), W = (uint32_t)threads / 32;
  const uint32_t rb = (nblk + W - 1) / W;
  // small tiles: 3 blocks per warp, 3 CTAs per SM; large tiles (level 7 Sierpinski: 69 blocks):
  // all 9 blocks' slots in registers (108 registers), 2 CTAs per SM (tools/packed_timing.py)
  if (p.dmax <= 5) {
    if (rb <= 3) return conway ? k_step_packed<5, true, 3, 256, 3, SH, BD, false> : k_step_packed<5, false, 3, 256, 3, SH, BD, false>;
    return conway ? k_step_packed<5, true, 9, 256, 2, SH, BD, false> : k_step_packed<5, false, 9, 256, 2, SH, BD, false>;
  }
  // one CTA per SM (the compacted-gather chunks of level-4 carpet tiles): 16 warps
  if (threads == 512 && BD && packed_compact_gathers(p) && !(p.pflags & kPackStaticItems))
    return conway ? k_step_packed<8, true, 6, 512, 1, SH, BD, BD> : k_step_packed<8, false, 6, 512, 1, SH, BD, BD>;
  if (threads == 512) return conway ? k_step_packed<8, true, 6, 512, 1, SH, BD, false> : k_step_packed<8, false, 6, 512, 1, SH, BD, false>;
  const bool dyn = BD && packed_compact_gathers(p) && !(p.pflags & kPackStaticItems);
  if (rb <= 2) {
    if (dyn) return conway ? k_step_packed<8, true, 2, 256, 3, SH, BD, BD> : k_step_packed<8, false, 2, 256, 3, SH, BD, BD>;
    return conway ? k_step_packed<8, true, 2, 256, 3, SH, BD, false> : k_step_packed<8, false, 2, 256, 3, SH, BD, false>;
  }
  if (dyn) return conway ? k_step_packed<8, true, 6, 256, 2, SH, BD, BD> : k_step_packed<8, false, 6, 256, 2, SH, BD, BD>;
  return conway ? k_step_packed<8, true, 6, 256, 2, SH, BD, false> : k_step_packed<8, false, 6, 256, 2, SH, BD, false>;
}

// link work by (direction, lane group) pairs when directions carry several links each
// (tools/packed_timing.py: carpet and empty bottles 20-23% faster, Sierpinski 6% slower)
static bool links_by_direction(const TileParams& p) { return p.E >= 3 * p.ndirs; }

template <bool SH>
static PackedFn pick_packed_s(const TileParams& p, int threads) {
  return links_by_direction(p) ? pick_packed_t<SH, true>(p, threads) : pick_packed_t<SH, false>(p, threads);
}

// SHARDED variants also read another shard's cells from the halo receive buffer.
static PackedFn pick_packed(const TileParams& p, int threads) {
  return p.halo.nneeds != 0 ? pick_packed_s<true>(p, threads) : pick_packed_s<false>(p, threads);
}

cudaError_t packed_prepare(const TileParams& p, size_t smem, int threads, int* occupancy) {
  cudaError_t e = cudaSuccess;
  for (PackedFn fn : {pick_packed_s<false>(p, threads), pick_packed_s<true>(p, threads)}) {
    e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick_packed_s<false>(p, threads), threads, smem);
  if (e != cudaSuccess) return e;
  *occupancy = blocks;
  return blocks > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t launch_step_packed(const TileParams& p, const uint32_t* cur, uint32_t* next, int grid, int threads,
                               size_t smem, cudaStream_t st) {
  if (pack_chunks(p) == 0) return cudaSuccess;
  pick_packed(p, threads)<<<grid, threads, smem, st>>>(p, reinterpret_cast<const uint4*>(cur),
                                                      reinterpret_cast<uint4*>(next));
  return cudaGetLastError();
}

static unsigned warps_grid(uint64_t warps) {
  uint64_t blocks = (warps + 7) / 8;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  return (unsigned)(blocks ? blocks : 1);
}

cudaError_t launch_pack(const TileParams& p, const uint8_t* st, uint32_t* packed, cudaStream_t s) {
  if (pack_chunks(p) == 0) return cudaSuccess;
  k_pack<<<warps_grid(pack_chunks(p) * 4 * ((p.Kw + 31) / 32)), 256, 0, s>>>(p, st, packed);
  return cudaGetLastError();
}

cudaError_t launch_unpack(const TileParams& p, const uint32_t* packed, uint8_t* st, cudaStream_t s) {
  if (pack_chunks(p) == 0) return cudaSuccess;
  k_unpack<<<warps_grid(pack_chunks(p) * 4 * ((p.Kp / 16 + 1) / 2)), 256, 0, s>>>(p, packed, st);
  return cudaGetLastError();
}

cudaError_t launch_seed_packed(const TileParams& p, const LevelMaps& full, uint32_t* packed, uint64_t seed, uint64_t q,
                               cudaStream_t s) {
  if (pack_chunks(p) == 0) return cudaSuccess;
  uint64_t z = seed;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  k_seed_packed<<<warps_grid(pack_chunks(p) * 4 * p.Kw), 256, 0, s>>>(p, full, packed, z, q);
  return cudaGetLastError();
}

cudaError_t launch_halo_pack_packed(const uint32_t* cur, const uint64_t* send_bits, uint64_t nsends, uint8_t* out,
                                   cudaStream_t st) {
  if (nsends == 0) return cudaSuccess;
  uint64_t blocks = (nsends + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  k_halo_pack_packed<<<(unsigned)blocks, 256, 0, st>>>(cur, send_bits, nsends, out);
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
