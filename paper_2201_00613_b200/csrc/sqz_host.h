// sqz_host.h — host-side planner of the Squeeze hot path (pure C++, no CUDA).
//
//  * spec validation and built-in replica tables
//  * checked geometry: V = k^r, compact k^⌊r/2⌋ x k^⌈r/2⌉, n = s^r
//  * the multi-digit λ/ν lookup tables of sqz_common.h for any level
//  * the level-g tile tables of the bit-sliced tile kernel: one
//    intra-tile neighbour table shared by every tile, plus the tile-boundary links
//  * contiguous chunk-aligned shard ranges and the halo plan
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "sqz_common.h"

namespace sqz {

struct Spec {
  uint32_t k = 0, s = 0;
  std::vector<uint8_t> tau;  // 2k: tau[2b] = τ_x(b), tau[2b+1] = τ_y(b)
  std::vector<int> hnu;      // s*s: hnu[ty*s + tx] = replica id or -1 (HOLE, reading D5)
};

// Returns 0 on success, else a squeeze_status code.
int make_spec(uint32_t k, uint32_t s, const uint8_t* tau, Spec& out);
bool builtin_spec(const std::string& name, uint32_t& k, uint32_t& s, std::vector<uint8_t>& tau);

FastDiv64 make_fastdiv(uint64_t d);

// Checked powers: return false on overflow past `limit`.
bool checked_pow(uint64_t base, uint32_t e, uint64_t limit, uint64_t& out);

struct HostLevelMaps {
  std::vector<uint32_t> lam_full, lam_tail, nu_full, nu_tail;
  LevelMaps view;  // host pointers into the vectors above
};
void build_level_maps(const Spec& f, uint32_t L, HostLevelMaps& out);

struct TileTables {
  uint32_t g = 0;
  uint64_t K = 1;          // k^g
  uint64_t h = 1;          // s^g
  uint32_t E = 0;          // distinct remote (direction, neighbour cell) words per tile
  uint32_t zero_slot = 0;  // index of the always-zero word in Z (= K + E)
  uint32_t max_degree = 0;
  uint32_t ndirs = 0;
  int dir_dx[8] = {0}, dir_dy[8] = {0};
  std::vector<uint16_t> nbr;       // K*8 indices into Z = [state words 0..K) | remote words | zero]
  std::vector<uint32_t> link_j;    // E: (first) own local cell touching it
  std::vector<uint32_t> link_j2;   // E: local cell inside the neighbour tile
  std::vector<uint8_t> link_dir;   // E: index into dir_dx/dir_dy (links sorted by direction)
  std::vector<uint16_t> dir_start; // ndirs + 1: links of direction d are [dir_start[d], dir_start[d+1])
  std::vector<uint32_t> local_x, local_y;  // K: λ_g(j)
};
// Builds the tables for level-g tiles.  Returns 0 or an error code.
int build_tile_tables(const Spec& f, uint32_t g, TileTables& t);

// Reorders the first D slots of every row (K rows x 8 word slots; the step sums them, so any
// order is correct) so that, for each group of 8 consecutive rows (the 8 lanes a 128-bit shared
// load serves per wavefront), the words each slot index reads fall on distinct 16-byte bank
// groups (word mod 8) as often as possible: fewer bank-conflict replays of the neighbour loads
// (DESIGN.md §5.1b).  Coordinate descent over the lanes (all permutations for D <= 5, swaps
// otherwise); deterministic.
void optimize_slot_order(std::vector<uint16_t>& rows, uint64_t K, int D);

// Largest g <= r with k^g <= max_cells and s^(2g) <= 1<<20 (auto tile level).
uint32_t auto_tile_level(const Spec& f, uint32_t r, uint64_t max_cells);

struct ShardRange {
  uint64_t tile_lo, tile_hi, omega_lo, omega_hi;
};
ShardRange shard_range(uint64_t num_tiles, uint64_t K, uint32_t rank, uint32_t nranks);

// Sorted unique Ω outside [tile_lo*K, tile_hi*K) that a cell inside has as a member
// neighbour.  coarse = level r-g maps; threads = worker threads.
void halo_needs(const TileTables& t, const LevelMaps& coarse, const ShardRange& sr,
                std::vector<uint64_t>& out, unsigned threads);

}  // namespace sqz
