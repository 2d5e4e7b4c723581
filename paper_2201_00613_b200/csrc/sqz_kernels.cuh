// sqz_kernels.cuh — kernel parameter blocks and launcher declarations (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_common.h"

namespace sqz {

// Tile-padded state layout (include/squeeze.h): cell Ω = t·K + j of this shard lives at byte
// (t - tile_lo)·Kp + j of a state buffer.
struct PadLayout {
  uint64_t tile_lo;
  uint64_t ntiles;   // local tiles
  uint32_t K, Kp;
  FastDiv64 divK;    // division by K
  FastDiv64 divKp;   // division by Kp
};

struct HaloView {
  uint64_t omega_lo, omega_hi;  // this shard
  PadLayout L;
  const uint64_t* needs;        // sorted Ω outside the shard
  uint64_t nneeds;
  const uint8_t* recv;          // recv[i] = state of needs[i]
  int* err;                     // set to 1 on a halo miss
};

struct TileParams {
  LevelMaps coarse;  // maps at level r - g (tile coordinates)
  uint64_t K;        // cells per tile
  uint32_t Kp;       // bytes per tile in a state buffer (K rounded up to 16)
  uint32_t St;       // bytes per tile slot in shared memory (odd multiple of 16, >= round_up(K, 32))
  uint32_t Kw;       // words per chunk in the packed layout (K rounded up to 4)
  uint32_t E;        // remote links per tile
  uint32_t zslot;    // index of the zero word in Z
  uint32_t dmax;     // max neighbour entries per cell
  uint32_t ndirs;
  uint32_t dir_code;  // 4 bits per direction d: (dx+1) | (dy+1) << 2
  const uint16_t* nbr;       // K*8
  const uint32_t* link_j2;   // E
  const uint8_t* link_dir;   // E (sorted by direction)
  const uint16_t* dir_start; // ndirs + 1
  uint64_t tile_lo, tile_hi, nchunks;
  uint32_t birth, survive;
  HaloView halo;
  // peer-memory halo (sqz_tile.cu epilogue): send entries of chunk c are
  // [peer_chunk_start[c], peer_chunk_start[c+1]); entry e stores byte (tile << 16 | j) of the
  // chunk's output into peer_recv[peer_of[e]][peer_pos[e]] (IPC-mapped receive buffers).
  uint8_t* const* peer_recv;
  const uint32_t* peer_chunk_start;
  const uint32_t* peer_cell;
  const uint32_t* peer_of;
  const uint64_t* peer_pos;
  // tile adjacency, built once at init: adj[d * adj_stride + (t - tile_lo)] = neighbour tile of
  // local tile t in link direction d, plus 1 (0 = none)
  const uint32_t* adj;
  uint64_t adj_stride;  // a multiple of kPackTiles
  uint32_t pstages;     // pipeline stages of the packed step
  uint32_t sin;        // input slice-ring depth of the large-tile byte step (sqz_stream.cu)
  uint32_t rcap;       // packed step, link items with E > kMaxPrefetchLinks: words of the compacted
                       // gather buffer (0 otherwise; sqz_packed.cu)
  uint32_t srcap;      // large-tile byte step: words of its compacted gather buffer (0: [32][E]; sqz_stream.cu)
  uint32_t pflags;     // packed step options (sqz_packed.cu kPack* flags; tuning A/B only)
};

// ν as an integer tensor-core product (sqz_mma.cu, SURVEY NEXT-3 ablation).
constexpr uint32_t kMmaMaxS2 = 256;  // s^2 <= 256 (H_ν staged in shared memory), k <= 256 (u8 A)
struct MmaNuParams {
  uint32_t r, s, k;
  uint32_t s_log2;       // log2 s if s is a power of two, else 0
  uint64_t n;            // s^r
  const int16_t* hnu;    // s*s: H_ν[θy * s + θx] or -1 (hole)
  const uint8_t* B;      // 32 x 8: B[μ-1][b] = byte b of k^(μ-1) (0 for μ > r)
};
cudaError_t launch_map_nu_mma(const MmaNuParams& q, const uint32_t* x, const uint32_t* y, uint64_t* om,
                              uint64_t count, cudaStream_t st);

// Shared-memory bytes the tile kernel needs for these parameters.
size_t tile_smem_bytes(const TileParams& p);
// Sets the shared-memory attribute of the kernel variant `p` selects and returns its
// occupancy (CTAs per SM) at `threads` threads.
cudaError_t tile_prepare(const TileParams& p, size_t smem, int threads, int* occupancy);

cudaError_t launch_lambda_engine(const LevelMaps& m, const uint8_t* cur, uint8_t* next, uint32_t birth,
                                 uint32_t survive, cudaStream_t st);
cudaError_t launch_block_step(const LevelMaps& coarse, uint32_t rho, const uint8_t* micro, uint32_t birth,
                              uint32_t survive, const uint8_t* cur, uint8_t* next, cudaStream_t st);
cudaError_t launch_block_seed(const LevelMaps& coarse, uint32_t rho, const uint8_t* micro, uint8_t* blocks,
                              uint64_t seed, uint64_t q, cudaStream_t st);
cudaError_t launch_tile_adjacency(const TileParams& p, uint32_t* adj, cudaStream_t st);
// Large-tile byte step (sqz_stream.cu): plan (ring depths, CTAs per SM), prepare, launch.
size_t stream_smem_bytes(const TileParams& p, bool peer);
bool stream_plan(TileParams& p, bool peer, int* minb);
int stream_threads();
cudaError_t stream_prepare(const TileParams& p, size_t smem, int minb, int* occupancy);
cudaError_t launch_step_stream(const TileParams& p, const uint8_t* cur, uint8_t* next, int grid, int minb,
                               size_t smem, cudaStream_t st);
size_t packed_smem_bytes(const TileParams& p);
// true when the packed step gathers out-of-chunk links through a compacted buffer of p.rcap words
bool packed_compact_gathers(const TileParams& p);
// false when the packed step's link work items would overflow (sqz_packed.cu); dir_start on the host
bool packed_items_fit(const uint16_t* dir_start, uint32_t ndirs, uint32_t E, uint32_t nwarps);
cudaError_t packed_prepare(const TileParams& p, size_t smem, int threads, int* occupancy);
cudaError_t launch_step_packed(const TileParams& p, const uint32_t* cur, uint32_t* next, int grid, int threads,
                               size_t smem, cudaStream_t st);
cudaError_t launch_pack(const TileParams& p, const uint8_t* st, uint32_t* packed, cudaStream_t s);
cudaError_t launch_unpack(const TileParams& p, const uint32_t* packed, uint8_t* st, cudaStream_t s);
cudaError_t launch_seed_packed(const TileParams& p, const LevelMaps& full, uint32_t* packed, uint64_t seed, uint64_t q,
                               cudaStream_t s);
cudaError_t launch_count_packed(const uint32_t* w, uint64_t nwords, uint64_t* out, cudaStream_t s);

cudaError_t launch_map_lambda(const LevelMaps& m, const uint64_t* om, uint32_t* x, uint32_t* y, uint64_t count,
                              cudaStream_t st);
cudaError_t launch_map_nu(const LevelMaps& m, const uint32_t* x, const uint32_t* y, uint64_t* om, uint64_t count,
                          cudaStream_t st);
cudaError_t launch_seed(const LevelMaps& m, const PadLayout& L, uint8_t* state, uint64_t seed, uint64_t q,
                        cudaStream_t st);
cudaError_t launch_step_naive(const LevelMaps& m, const uint8_t* cur, uint8_t* next, uint32_t birth, uint32_t survive,
                              const HaloView& halo, cudaStream_t st);
cudaError_t launch_step_tile(const TileParams& p, const uint8_t* cur, uint8_t* next, int grid, int threads,
                             size_t smem, cudaStream_t st);
cudaError_t launch_count_alive(const uint8_t* state, uint64_t bytes, uint64_t* out, cudaStream_t st);
cudaError_t launch_halo_peer_push(const uint8_t* cur, const uint64_t* send_offsets, const uint32_t* send_peer,
                                  const uint64_t* send_pos, uint64_t nsends, uint8_t* const* peer_recv, cudaStream_t st);
cudaError_t launch_halo_pack_packed(const uint32_t* cur, const uint64_t* send_bits, uint64_t nsends, uint8_t* out,
                                   cudaStream_t st);
cudaError_t launch_halo_pack(const uint8_t* cur, const uint64_t* send_offsets, uint64_t nsends, uint8_t* out,
                             cudaStream_t st);
cudaError_t launch_bb_seed(const LevelMaps& m, uint8_t* grid, uint64_t seed, uint64_t q, cudaStream_t st);
cudaError_t launch_bb_step(const uint8_t* cur, uint8_t* next, uint64_t n, uint32_t birth, uint32_t survive,
                           cudaStream_t st);
// bit-sliced BB step (sqz_bb.cu) for n % 32 == 0
bool bb_bits_ok(uint64_t n);
cudaError_t launch_bb_step_bits(const uint8_t* cur, uint8_t* next, uint64_t n, uint32_t birth, uint32_t survive,
                                cudaStream_t st);
cudaError_t launch_bb_to_compact(const LevelMaps& m, const PadLayout& L, const uint8_t* grid, uint8_t* state,
                                 cudaStream_t st);

}  // namespace sqz
