// sqz_api.cu — the extern "C" boundary declared in include/squeeze.h.
//
// Owns the context (host planner state + device copies of the tables) and dispatches to
// the kernels of sqz_kernels.cu.  No C++ exception crosses the boundary: every entry
// point is wrapped and returns a squeeze_status.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/squeeze.h"
#include "sqz_host.h"
#include "sqz_heat.cuh"
#include "sqz_kernels.cuh"

using namespace sqz;

namespace {

struct DeviceLUTs {
  uint32_t* d = nullptr;
  LevelMaps view{};
};

// Block-level Squeeze at rho = s^m: maps at level r - m and the rho x rho micro-fractal mask.
struct BlockLevel {
  HostLevelMaps host;
  DeviceLUTs dev;
  uint8_t* d_micro = nullptr;
};

struct Ctx {
  Spec f;
  uint32_t r = 0;
  squeeze_rule rule{};
  uint32_t rank = 0, nranks = 1;
  squeeze_options opts{};
  uint64_t V = 1, n = 1, cw = 1, ch = 1;
  HostLevelMaps full, coarse;
  TileTables tt;
  uint64_t NT = 1;
  ShardRange sr{};
  uint64_t state_bytes = 0;
  uint32_t Kp = 16;  // bytes per tile in a state buffer (tile-padded layout)
  std::vector<uint64_t> needs, sends, send_offsets;
  std::vector<uint64_t> send_bits;  // packed layout: u32 index << 5 | bit of each send cell
  // device
  int device = -1;
  DeviceLUTs d_full, d_coarse;
  uint16_t* d_nbr = nullptr;
  uint16_t* d_nbr_packed = nullptr;  // neighbour slots for the packed kernel (links after Kw words)
  uint32_t* d_adj = nullptr;         // tile adjacency [ndirs][local tiles], built once at init
  int packed_threads = 256;
  uint32_t packed_stages = 3;
  uint32_t packed_rcap = 0;  // compacted link-gather buffer of the packed step (words; 0 = none)
  uint32_t packed_flags = 0;  // packed step options (sqz_packed.cu kPack*; A/B knobs)
  uint32_t Kw = 4;                    // packed words per chunk
  uint64_t packed_bytes = 0;
  int packed_grid = 0;
  size_t packed_smem = 0;
  // heat workload (NEXT-4): neighbour slots, remote pairs, launch shape
  uint32_t heat_P = 0, heat_stages = 3;
  uint64_t heat_bytes = 0;
  int heat_grid = 0;
  uint16_t* d_heat_nbr = nullptr;
  uint32_t* d_heat_pairs = nullptr;
  uint32_t* d_heat_j2 = nullptr;
  int16_t* d_mma_h = nullptr;   // ν tensor-core ablation tables (NEXT-3)
  uint8_t* d_mma_B = nullptr;
  uint32_t* d_link_j2 = nullptr;
  uint8_t* d_link_dir = nullptr;
  uint16_t* d_dir_start = nullptr;
  uint64_t* d_needs = nullptr;
  uint64_t* d_sends = nullptr;
  uint64_t* d_send_bits = nullptr;
  // peer-memory halo: per-chunk CSR of the send cells and their destinations (squeeze_halo_peer_*)
  uint32_t* d_peer_chunk_start = nullptr;
  uint32_t* d_peer_cell = nullptr;
  uint32_t* d_peer_of = nullptr;
  uint64_t* d_peer_pos = nullptr;
  uint8_t** d_peer_recv[2] = {nullptr, nullptr};
  uint32_t* d_send_peer = nullptr;  // the same destinations in send order (squeeze_halo_peer_push)
  uint64_t* d_send_pos = nullptr;
  int peer_parity = -1;  // -1: fused stores off
  uint32_t peer_slots[2] = {0, 0};  // entries of the bound peer pointer arrays (== nranks)
  int* d_err = nullptr;
  uint8_t* d_send = nullptr;
  const uint8_t* d_recv = nullptr;
  int tile_threads = 0, tile_grid = 0;
  size_t tile_smem = 0;
  // large tiles (a 32-tile chunk does not fit shared memory twice): the streaming byte step
  bool stream = false;
  int stream_minb = 1, stream_grid = 0;
  uint32_t stream_sin = 0;
  uint32_t stream_srcap = 0;  // compacted gather buffer of the streaming step (words; 0 = [32][E])
  std::map<uint32_t, BlockLevel> blocks;  // by m = log_s rho
  // CUDA graph of the two-step ping-pong
  cudaGraphExec_t graph = nullptr;
  const uint8_t* graph_a = nullptr;
  const uint8_t* graph_b = nullptr;
  cudaStream_t graph_stream = nullptr;
};

struct DevGuard {
  int prev = -1;
  bool active = false;
  explicit DevGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      cudaSetDevice(dev);
      active = true;
    }
  }
  ~DevGuard() {
    if (active) cudaSetDevice(prev);
  }
};

squeeze_status cu(cudaError_t e) { return e == cudaSuccess ? SQZ_OK : SQZ_E_CUDA; }

template <class T>
squeeze_status upload(T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return SQZ_OK;
  if (cudaMalloc((void**)dst, n * sizeof(T)) != cudaSuccess) return SQZ_E_NOMEM;
  return cu(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
}

squeeze_status upload_maps(const HostLevelMaps& h, DeviceLUTs& d) {
  size_t n0 = h.lam_full.size(), n1 = h.lam_tail.size(), n2 = h.nu_full.size(), n3 = h.nu_tail.size();
  std::vector<uint32_t> all;
  all.reserve(n0 + n1 + n2 + n3);
  all.insert(all.end(), h.lam_full.begin(), h.lam_full.end());
  all.insert(all.end(), h.lam_tail.begin(), h.lam_tail.end());
  all.insert(all.end(), h.nu_full.begin(), h.nu_full.end());
  all.insert(all.end(), h.nu_tail.begin(), h.nu_tail.end());
  squeeze_status st = upload(&d.d, all.data(), all.size());
  if (st != SQZ_OK) return st;
  d.view = h.view;
  d.view.lam_full = d.d;
  d.view.lam_tail = d.d + n0;
  d.view.nu_full = d.d + n0 + n1;
  d.view.nu_tail = d.d + n0 + n1 + n2;
  return SQZ_OK;
}

void free_device(Ctx* c) {
  if (c->device < 0) return;
  DevGuard g(c->device);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  cudaFree(c->d_full.d);
  cudaFree(c->d_coarse.d);
  cudaFree(c->d_nbr);
  cudaFree(c->d_nbr_packed);
  cudaFree(c->d_heat_nbr);
  cudaFree(c->d_mma_h);
  cudaFree(c->d_mma_B);
  cudaFree(c->d_heat_pairs);
  cudaFree(c->d_heat_j2);
  cudaFree(c->d_adj);
  for (auto& kv : c->blocks) {
    cudaFree(kv.second.dev.d);
    cudaFree(kv.second.d_micro);
  }
  cudaFree(c->d_link_j2);
  cudaFree(c->d_link_dir);
  cudaFree(c->d_dir_start);
  cudaFree(c->d_needs);
  cudaFree(c->d_send_bits);
  cudaFree(c->d_peer_chunk_start);
  cudaFree(c->d_peer_cell);
  cudaFree(c->d_peer_of);
  cudaFree(c->d_peer_pos);
  cudaFree(c->d_send_peer);
  cudaFree(c->d_send_pos);
  cudaFree(c->d_peer_recv[0]);
  cudaFree(c->d_peer_recv[1]);
  cudaFree(c->d_sends);
  cudaFree(c->d_err);
}

PadLayout pad_layout(const Ctx* c) {
  PadLayout L;
  L.tile_lo = c->sr.tile_lo;
  L.ntiles = c->sr.tile_hi - c->sr.tile_lo;
  L.K = (uint32_t)c->tt.K;
  L.Kp = c->Kp;
  L.divK = make_fastdiv(c->tt.K);
  L.divKp = make_fastdiv(c->Kp);
  return L;
}

HaloView halo_view(const Ctx* c) {
  HaloView h;
  h.L = pad_layout(c);
  h.omega_lo = c->sr.omega_lo;
  h.omega_hi = c->sr.omega_hi;
  h.needs = c->d_needs;
  h.nneeds = c->needs.size();
  h.recv = c->d_recv;
  h.err = c->d_err;
  return h;
}

squeeze_status check_state(const Ctx* c, const void* p) {
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  if (c->state_bytes == 0 && p == nullptr) return SQZ_OK;  // empty shard: every call is a no-op
  if (p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u)) return SQZ_E_CONFIG;
  return SQZ_OK;
}

// Rows of the adjacency table are padded to whole packed chunks (the packed kernel bulk-copies them).
uint64_t adj_stride(const Ctx* c) {
  return (c->sr.tile_hi - c->sr.tile_lo + kPackTiles - 1) / kPackTiles * kPackTiles;
}

TileParams tile_params(const Ctx* c) {
  TileParams p{};
  p.coarse = c->d_coarse.view;
  p.K = c->tt.K;
  p.Kp = c->Kp;
  p.St = c->Kp;
  p.E = c->tt.E;
  p.zslot = c->tt.zero_slot;
  p.dmax = c->tt.max_degree;
  p.ndirs = c->tt.ndirs;
  p.dir_code = 0;
  for (uint32_t i = 0; i < c->tt.ndirs; ++i)
    p.dir_code |= (uint32_t)((c->tt.dir_dx[i] + 1) | ((c->tt.dir_dy[i] + 1) << 2)) << (4 * i);
  p.nbr = c->d_nbr;
  p.link_j2 = c->d_link_j2;
  p.link_dir = c->d_link_dir;
  p.dir_start = c->d_dir_start;
  p.tile_lo = c->sr.tile_lo;
  p.tile_hi = c->sr.tile_hi;
  p.nchunks = (c->sr.tile_hi - c->sr.tile_lo + kChunkTiles - 1) / kChunkTiles;
  p.birth = c->rule.birth_mask;
  p.survive = c->rule.survive_mask;
  p.Kw = c->Kw;
  p.halo = halo_view(c);
  p.adj = c->d_adj;
  p.adj_stride = adj_stride(c);
  p.pstages = c->packed_stages;
  p.rcap = c->packed_rcap;
  p.pflags = c->packed_flags;
  p.sin = c->stream_sin;
  p.srcap = c->stream_srcap;
  if (c->peer_parity >= 0 && c->d_peer_chunk_start) {
    p.peer_recv = c->d_peer_recv[c->peer_parity];
    p.peer_chunk_start = c->d_peer_chunk_start;
    p.peer_cell = c->d_peer_cell;
    p.peer_of = c->d_peer_of;
    p.peer_pos = c->d_peer_pos;
  }
  return p;
}

HeatParams heat_params(const Ctx* c, float alpha) {
  HeatParams h{};
  h.K = (uint32_t)c->tt.K;
  h.P = c->heat_P;
  h.stages = c->heat_stages;
  h.alpha = alpha;
  h.nbr = c->d_heat_nbr;
  h.pairs = c->d_heat_pairs;
  h.pair_j2 = c->d_heat_j2;
  return h;
}

squeeze_status do_heat_step(Ctx* c, const float* cur, float* next, float alpha, cudaStream_t st) {
  if (c->nranks > 1) return SQZ_E_CONFIG;
  if (c->NT >= 0xFFFFFFFFull) return SQZ_E_OVERFLOW;
  if (c->heat_grid == 0) return SQZ_E_INVALID_LEVEL;  // the heat unit does not fit at this tile level
  return cu(launch_heat_step(heat_params(c, alpha), tile_params(c), cur, next, c->heat_grid, st));
}

squeeze_status do_step(Ctx* c, const uint8_t* cur, uint8_t* next, cudaStream_t st) {
  if (c->nranks > 1 && !c->needs.empty() && c->d_recv == nullptr) return SQZ_E_CONFIG;
  if (c->NT >= 0xFFFFFFFFull) return SQZ_E_OVERFLOW;  // the tile kernel keeps tile indices in 32 bits
  TileParams p = tile_params(c);
  if (c->stream) {
    int grid = (int)std::min<uint64_t>((uint64_t)c->stream_grid, p.nchunks ? p.nchunks : 1);
    return cu(launch_step_stream(p, cur, next, grid, c->stream_minb, c->tile_smem, st));
  }
  int grid = (int)std::min<uint64_t>((uint64_t)c->tile_grid, p.nchunks ? p.nchunks : 1);
  return cu(launch_step_tile(p, cur, next, grid, c->tile_threads, c->tile_smem, st));
}

squeeze_status do_step_packed(Ctx* c, const uint32_t* cur, uint32_t* next, cudaStream_t st) {
  if (c->nranks > 1 && !c->needs.empty() && c->d_recv == nullptr) return SQZ_E_CONFIG;
  if (c->NT >= 0xFFFFFFFFull) return SQZ_E_OVERFLOW;
  if (c->packed_grid == 0) return SQZ_E_INVALID_LEVEL;  // the packed chunk does not fit at this tile level
  TileParams p = tile_params(c);
  p.nbr = c->d_nbr_packed;
  const uint64_t pch = (p.tile_hi - p.tile_lo + kPackTiles - 1) / kPackTiles;
  int grid = (int)std::min<uint64_t>((uint64_t)c->packed_grid, pch ? pch : 1);
  return cu(launch_step_packed(p, cur, next, grid, c->packed_threads, c->packed_smem, st));
}

// m = log_s rho, or -1 if rho is not a power of s (or exceeds the level / 32).
int block_m(const Ctx* c, uint32_t rho) {
  uint64_t v = 1;
  for (int m = 0; m <= (int)c->r; ++m) {
    if (v == rho) return (rho <= 32) ? m : -1;
    v *= c->f.s;
  }
  return -1;
}

squeeze_status block_level(Ctx* c, uint32_t rho, BlockLevel** out) {
  const int m = block_m(c, rho);
  if (m < 0) return SQZ_E_INVALID_LEVEL;
  auto it = c->blocks.find((uint32_t)m);
  if (it == c->blocks.end()) {
    BlockLevel bl;
    build_level_maps(c->f, c->r - (uint32_t)m, bl.host);
    HostLevelMaps micro_maps;
    build_level_maps(c->f, (uint32_t)m, micro_maps);
    std::vector<uint8_t> mask((size_t)rho * rho);
    for (uint32_t y = 0; y < rho; ++y)
      for (uint32_t x = 0; x < rho; ++x) mask[(size_t)y * rho + x] = nu_level(micro_maps.view, x, y) != kNoneU64;
    squeeze_status st = upload_maps(bl.host, bl.dev);
    if (st == SQZ_OK) st = upload(&bl.d_micro, mask.data(), mask.size());
    if (st != SQZ_OK) return st;
    bl.dev.view = bl.host.view;  // re-point the view at the device copies
    bl.dev.view.lam_full = bl.dev.d;
    bl.dev.view.lam_tail = bl.dev.d + bl.host.lam_full.size();
    bl.dev.view.nu_full = bl.dev.d + bl.host.lam_full.size() + bl.host.lam_tail.size();
    bl.dev.view.nu_tail = bl.dev.view.nu_full + bl.host.nu_full.size();
    it = c->blocks.emplace((uint32_t)m, std::move(bl)).first;
  }
  *out = &it->second;
  return SQZ_OK;
}

template <class F>
squeeze_status guarded(F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return SQZ_E_NOMEM;
  } catch (...) {
    return SQZ_E_CONFIG;
  }
}

}  // namespace

extern "C" {

const char* squeeze_version(void) { return "squeeze-b200 0.1 (sm_100a)"; }

const char* squeeze_strerror(squeeze_status st) {
  switch (st) {
    case SQZ_OK: return "ok";
    case SQZ_E_INVALID_SPEC: return "invalid fractal spec (S:29-33 invariants)";
    case SQZ_E_OVERFLOW: return "level too large: s^r > 2^32 or k^r >= 2^62";
    case SQZ_E_OUT_OF_BOUNDS: return "coordinate out of bounds";
    case SQZ_E_HOLE: return "coordinate is a hole of the fractal";
    case SQZ_E_INVALID_LEVEL: return "invalid level or tile level";
    case SQZ_E_CONFIG: return "invalid configuration or argument";
    case SQZ_E_CUDA: return "CUDA runtime error";
    case SQZ_E_NO_DEVICE: return "host-only context: no device bound";
    case SQZ_E_NOMEM: return "out of memory";
    case SQZ_E_HALO: return "halo plan missed a needed out-of-shard neighbour";
  }
  return "unknown status";
}

squeeze_status squeeze_builtin_fractal(const char* name, uint32_t* k, uint32_t* s, uint8_t* tau_out, uint32_t cap) {
  return guarded([&]() -> squeeze_status {
    if (!name || !k || !s) return SQZ_E_CONFIG;
    std::vector<uint8_t> tau;
    if (!builtin_spec(name, *k, *s, tau)) return SQZ_E_INVALID_SPEC;
    if (tau_out) {
      if (cap < tau.size()) return SQZ_E_CONFIG;
      std::memcpy(tau_out, tau.data(), tau.size());
    }
    return SQZ_OK;
  });
}

squeeze_status squeeze_init(void** out_ctx, const squeeze_fractal* f, uint32_t r, const squeeze_rule* rule,
                            const squeeze_shard* shard, const squeeze_options* opts, int device) {
  return guarded([&]() -> squeeze_status {
    if (!out_ctx || !f) return SQZ_E_CONFIG;
    *out_ctx = nullptr;
    Ctx* c = new Ctx();
    auto fail = [&](squeeze_status st) {
      free_device(c);
      delete c;
      return st;
    };
    int rc = make_spec(f->k, f->s, f->tau, c->f);
    if (rc != SQZ_OK) return fail((squeeze_status)rc);
    c->r = r;
    c->rule = rule ? *rule : squeeze_rule{(uint16_t)(1u << 3), (uint16_t)((1u << 2) | (1u << 3))};
    if ((c->rule.birth_mask | c->rule.survive_mask) & ~0x1FFu) return fail(SQZ_E_CONFIG);
    if (shard) {
      if (shard->nranks == 0 || shard->rank >= shard->nranks) return fail(SQZ_E_CONFIG);
      c->rank = shard->rank;
      c->nranks = shard->nranks;
    }
    if (opts) c->opts = *opts;
    // checked geometry: coordinates fit 32 bits, Ω fits 62 bits
    if (!checked_pow(c->f.s, r, 1ull << 32, c->n) || !checked_pow(c->f.k, r, (1ull << 62) - 1, c->V))
      return fail(SQZ_E_OVERFLOW);
    checked_pow(c->f.k, r / 2, ~0ull, c->cw);
    checked_pow(c->f.k, (r + 1) / 2, ~0ull, c->ch);
    uint32_t g = c->opts.tile_level ? c->opts.tile_level : auto_tile_level(c->f, r, 1024);
    if (g > r) return fail(SQZ_E_INVALID_LEVEL);
    rc = build_tile_tables(c->f, g, c->tt);
    if (rc != SQZ_OK) return fail((squeeze_status)rc);
    // link-heavy fractals (more than 2% of a tile's cells are boundary links, e.g. the carpet's
    // full tile edges) take the next tile level when it has at most 4096 cells: links grow
    // with the tile perimeter, cells with k^g (SURVEY §7 hard part 3; the streaming byte step)
    if (!c->opts.tile_level && g < r && (uint64_t)c->tt.E * 50 > c->tt.K && c->tt.K * c->f.k <= 4096) {
      TileTables up;
      if (build_tile_tables(c->f, g + 1, up) == SQZ_OK) {
        c->tt = std::move(up);
        g = g + 1;
      }
    }
    build_level_maps(c->f, r, c->full);
    build_level_maps(c->f, r - g, c->coarse);
    checked_pow(c->f.k, r - g, ~0ull, c->NT);
    c->sr = shard_range(c->NT, c->tt.K, c->rank, c->nranks);
    // tile-padded layout: Kp >= round_up(K, 32) and Kp/16 odd, so the 128-bit lane accesses of
    // the tile kernel are bank-conflict-free (measured: 15.7 vs 16.1 ms at r=22 despite +2.2% bytes)
    c->Kp = (uint32_t)((c->tt.K + 31) & ~31ull);
    if ((c->Kp / 16) % 2 == 0) c->Kp += 16;
    {  // two double-buffered 32-tile chunks per SM, else the streaming step (sqz_stream.cu), whose
       // tiles are rows of round_up(K, 32) bytes (whole 32-cell blocks, 256-bit aligned stores)
      TileParams q{};
      q.K = c->tt.K;
      q.Kp = c->Kp;
      q.St = c->Kp;
      q.E = c->tt.E;
      q.ndirs = c->tt.ndirs;
      q.dmax = c->tt.max_degree;
      c->stream = 2 * tile_smem_bytes(q) > 227 * 1024;
      if (c->stream) c->Kp = (uint32_t)((c->tt.K + 31) & ~31ull);
    }
    c->state_bytes = (c->sr.tile_hi - c->sr.tile_lo) * c->Kp;
    c->Kw = (uint32_t)((c->tt.K + 3) & ~3ull);
    c->packed_bytes = ((c->sr.tile_hi - c->sr.tile_lo + kPackTiles - 1) / kPackTiles) * c->Kw * 16;
    c->heat_bytes = ((c->sr.tile_hi - c->sr.tile_lo + 3) / 4) * c->tt.K * 16;  // 4-tile float4 chunks
    if (c->nranks > 1) {
      unsigned th = std::max(1u, std::thread::hardware_concurrency());
      halo_needs(c->tt, c->coarse.view, c->sr, c->needs, th);
    }
    c->device = device;
    if (device >= 0) {
      DevGuard dg(device);
      if (cudaSetDevice(device) != cudaSuccess) return fail(SQZ_E_CUDA);
      squeeze_status st;
      if ((st = upload_maps(c->full, c->d_full)) != SQZ_OK) return fail(st);
      if ((st = upload_maps(c->coarse, c->d_coarse)) != SQZ_OK) return fail(st);
      // the tile kernel reads neighbour slots as byte offsets into its Z word array
      if ((uint64_t)c->tt.zero_slot * 4 > 0xFFFFu) return fail(SQZ_E_INVALID_LEVEL);
      std::vector<uint16_t> nbr_bytes(c->tt.nbr.size()), nbr_packed(c->tt.nbr.size());
      for (size_t i = 0; i < nbr_bytes.size(); ++i) {
        const uint32_t v = c->tt.nbr[i];
        nbr_bytes[i] = (uint16_t)(v * 4u);
        // packed kernel: word slots; state words fill [0, Kw), link words follow at Kw + e
        nbr_packed[i] = (uint16_t)(v < c->tt.K ? v : v - c->tt.K + c->Kw);
      }
      if ((uint64_t)(c->Kw + c->tt.E + 1) > 0xFFFFu) return fail(SQZ_E_INVALID_LEVEL);
      // 128-bit neighbour loads of the packed step: spread each quarter-warp's words over the
      // shared-memory bank groups (sqz_host.h optimize_slot_order)
      optimize_slot_order(nbr_packed, c->tt.K, c->tt.max_degree <= 5 ? 5 : 8);
      if ((st = upload(&c->d_nbr, nbr_bytes.data(), nbr_bytes.size())) != SQZ_OK) return fail(st);
      if ((st = upload(&c->d_nbr_packed, nbr_packed.data(), nbr_packed.size())) != SQZ_OK) return fail(st);
      if ((st = upload(&c->d_link_j2, c->tt.link_j2.data(), c->tt.link_j2.size())) != SQZ_OK) return fail(st);
      if ((st = upload(&c->d_link_dir, c->tt.link_dir.data(), c->tt.link_dir.size())) != SQZ_OK) return fail(st);
      if ((st = upload(&c->d_dir_start, c->tt.dir_start.data(), c->tt.dir_start.size())) != SQZ_OK) return fail(st);
      if ((st = upload(&c->d_needs, c->needs.data(), c->needs.size())) != SQZ_OK) return fail(st);
      if (cudaMalloc((void**)&c->d_err, sizeof(int)) != cudaSuccess) return fail(SQZ_E_NOMEM);
      if (cudaMemset(c->d_err, 0, sizeof(int)) != cudaSuccess) return fail(SQZ_E_CUDA);
      // tile kernel launch shape: persistent CTAs, threads ~ one per tile cell
      TileParams p{};
      p.K = c->tt.K;
      p.Kp = c->Kp;
      p.St = c->Kp;
      p.E = c->tt.E;
      p.ndirs = c->tt.ndirs;
      p.dmax = c->tt.max_degree;
      p.birth = c->rule.birth_mask;
      p.survive = c->rule.survive_mask;
      c->tile_smem = tile_smem_bytes(p);
      uint32_t threads = c->opts.block_threads;
      if (threads == 0) threads = 256;  // 8 warps, 3 CTAs per SM (tools/sweep.py)
      if (threads % 32 || threads > 1024) return fail(SQZ_E_CONFIG);
      c->tile_threads = (int)threads;
      int occ = 0;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      // two double-buffered 32-tile chunks per SM, else the streaming step (sqz_stream.cu)
      if (!c->stream && tile_prepare(p, c->tile_smem, c->tile_threads, &occ) != cudaSuccess) return fail(SQZ_E_INVALID_LEVEL);
      if (c->stream) {
        if (c->tt.K > 0xFFFFu || !stream_plan(p, c->nranks > 1, &c->stream_minb)) return fail(SQZ_E_INVALID_LEVEL);
        c->stream_sin = p.sin;
        c->stream_srcap = p.srcap;
        c->tile_smem = stream_smem_bytes(p, c->nranks > 1);
        c->tile_threads = stream_threads();
        const cudaError_t se = stream_prepare(p, c->tile_smem, c->stream_minb, &occ);
        if (getenv("SQZ_DEBUG"))
          fprintf(stderr, "sqz: streaming step K=%llu E=%u input ring %u smem %zu minb %d occupancy %d (%s)\n",
                  (unsigned long long)c->tt.K, c->tt.E, p.sin, c->tile_smem, c->stream_minb, occ,
                  cudaGetErrorString(se));
        if (se != cudaSuccess) return fail(SQZ_E_INVALID_LEVEL);
        c->stream_grid = sms * std::max(1, occ);
        if (const char* e = getenv("SQZ_STREAM_GRID"))  // tests: several chunks per CTA at small sizes
          if (atoi(e) > 0) c->stream_grid = std::min(c->stream_grid, atoi(e));
      }
      if (c->opts.ctas_per_sm) occ = std::min<int>(occ, (int)c->opts.ctas_per_sm);
      c->tile_grid = sms * std::max(1, occ);
      p.Kw = c->Kw;
      // packed step: 8 warps (tools/packed_timing.py: 8 warps with every block's slots in
      // registers beat 16 warps at 64 registers); 4 stages if three CTAs fit an SM, else 3 if
      // two do, else 2
      c->packed_threads = 256;
      // stages: 4 if three CTAs still fit an SM, else 3 if two do, else 2
      // A/B: the compacted link gathers (dynamic link items) for every link-item context (flag 4)
      if (const char* e = getenv("SQZ_PACKED_COMPACT"))
        if (atoi(e) && c->tt.E >= 3 * c->tt.ndirs) c->packed_flags |= 4u;
      p.pflags = c->packed_flags;
      p.pstages = 4;
      if (3 * packed_smem_bytes(p) > 220 * 1024) p.pstages = 3;
      if (p.pstages == 3 && 2 * packed_smem_bytes(p) > 220 * 1024) p.pstages = 2;
      if (const char* e = getenv("SQZ_PACKED_STAGES")) p.pstages = (uint32_t)atoi(e);
      if (p.pstages < 2 || p.pstages > 4) return fail(SQZ_E_CONFIG);
      // more links than the [tile][link] gather buffer holds (the carpet at level 4): a compacted
      // buffer of the outside (tile, link) pairs, as large as the CTAs per SM allow (at most every
      // pair of the chunk); pairs past it are read synchronously (sqz_packed.cu)
      p.rcap = 0;
      if (packed_compact_gathers(p)) {
        const size_t base = packed_smem_bytes(p), budget = 2 * base <= 200 * 1024 ? 110 * 1024 : 226 * 1024;
        if (base < budget) p.rcap = (uint32_t)std::min<size_t>((size_t)kPackTiles * p.E, (budget - base) / 4) & ~31u;
        if (const char* e = getenv("SQZ_PACKED_RCAP")) p.rcap = std::min<uint32_t>(p.rcap, (uint32_t)atoi(e));  // tests: overflow
      }
      c->packed_rcap = p.rcap;
      // A/B: the compacted gathers with the static link-item split (2) instead of the dynamic one
      if (const char* e = getenv("SQZ_PACKED_STATIC_ITEMS"))
        c->packed_flags = (c->packed_flags & ~2u) | (atoi(e) ? 2u : 0u);
      p.pflags = c->packed_flags;
      // a compacted-gather chunk leaves one CTA per SM: 16 warps instead of 8 (8 neighbour slots only)
      if (p.rcap && p.dmax > 5 && 2 * packed_smem_bytes(p) > 228 * 1024) c->packed_threads = 512;
      if (const char* e = getenv("SQZ_PACKED_THREADS"))  // A/B timing
        if (p.dmax > 5 && (atoi(e) == 256 || atoi(e) == 512)) c->packed_threads = atoi(e);
      c->packed_stages = p.pstages;
      c->packed_smem = packed_smem_bytes(p);
      int pocc = 0;
      // a chunk of 128 tiles that does not fit shared memory leaves the packed step unavailable at
      // this tile level (its entry points return SQZ_E_INVALID_LEVEL), not the context
      if (c->packed_smem <= 227 * 1024 &&
          packed_items_fit(c->tt.dir_start.data(), c->tt.ndirs, c->tt.E, (uint32_t)c->packed_threads / 32) &&
          packed_prepare(p, c->packed_smem, c->packed_threads, &pocc) == cudaSuccess)
        c->packed_grid = sms * std::max(1, pocc);
      else
        c->packed_grid = 0;
      if (const char* e = getenv("SQZ_PACKED_GRID"))  // tests: several chunks per CTA at small sizes
        if (atoi(e) > 0 && c->packed_grid) c->packed_grid = std::min(c->packed_grid, atoi(e));
      // ν tensor-core ablation: H_ν as int16 and the per-level weight bytes of k^(μ-1)
      if (c->f.s * c->f.s <= kMmaMaxS2 && c->f.k <= 256 && r <= 32) {
        std::vector<int16_t> hh(c->f.hnu.begin(), c->f.hnu.end());
        std::vector<uint8_t> B(32 * 8, 0);
        uint64_t w = 1;
        for (uint32_t m = 0; m < r; ++m) {
          for (int b = 0; b < 8; ++b) B[m * 8 + b] = (uint8_t)(w >> (8 * b));
          w *= c->f.k;
        }
        if ((st = upload(&c->d_mma_h, hh.data(), hh.size())) != SQZ_OK) return fail(st);
        if ((st = upload(&c->d_mma_B, B.data(), B.size())) != SQZ_OK) return fail(st);
      }
      // heat workload: slots = float4 words of a chunk's [K state | P pairs] shared slot; an
      // absent neighbour is the cell itself, a remote neighbour a per-(cell, link) pair
      {
        std::vector<uint16_t> hn(c->tt.nbr.size());
        std::vector<uint32_t> hp, hj2;
        for (uint64_t j = 0; j < c->tt.K; ++j)
          for (int k = 0; k < 8; ++k) {
            const uint32_t v = c->tt.nbr[j * 8 + k];
            uint64_t slot;
            if (v < c->tt.K) slot = v;
            else if (v == c->tt.zero_slot) slot = j;
            else {
              const uint32_t e = v - (uint32_t)c->tt.K;
              slot = c->tt.K + hp.size();
              hp.push_back((uint32_t)j | ((uint32_t)c->tt.link_dir[e] << 16));
              hj2.push_back(c->tt.link_j2[e]);
            }
            if (slot > 0xFFFFu) return fail(SQZ_E_INVALID_LEVEL);
            hn[j * 8 + k] = (uint16_t)slot;
          }
        c->heat_P = (uint32_t)hp.size();
        // the same 128-bit quarter-warp bank-group spreading as the packed table (the slot order
        // only changes the order of the float32 sum, inside the D16 bound)
        optimize_slot_order(hn, c->tt.K, c->tt.max_degree <= 5 ? 5 : 8);
        if ((st = upload(&c->d_heat_nbr, hn.data(), hn.size())) != SQZ_OK) return fail(st);
        if ((st = upload(&c->d_heat_pairs, hp.data(), hp.size())) != SQZ_OK) return fail(st);
        if ((st = upload(&c->d_heat_j2, hj2.data(), hj2.size())) != SQZ_OK) return fail(st);
        HeatParams h = heat_params(c, 0.125f);
        TileParams q = tile_params(c);
        for (c->heat_stages = 3; c->heat_stages > 2; --c->heat_stages) {  // 3 CTAs per SM if they fit
          h.stages = c->heat_stages;
          if (3 * heat_smem_bytes(h, q) <= 220 * 1024) break;
        }  // (at least 2 stages: a unit's successor is filled while the unit is computed)
        h.stages = c->heat_stages;
        int hocc = 0;
        // a heat unit that does not fit shared memory leaves the heat step unavailable at this tile
        // level (its calls return SQZ_E_INVALID_LEVEL); no attribute call is made for it
        c->heat_grid = heat_smem_bytes(h, q) <= 227 * 1024 && heat_prepare(h, q, &hocc) == cudaSuccess
                           ? sms * std::max(1, hocc) : 0;
      }
      // tile adjacency: the coarse λ and one coarse ν per link direction of every local tile,
      // evaluated once here instead of every step
      const uint64_t ntl = c->sr.tile_hi - c->sr.tile_lo;
      if (ntl && c->tt.ndirs && c->NT < 0xFFFFFFFFull) {
        const size_t adj_bytes = adj_stride(c) * c->tt.ndirs * sizeof(uint32_t);
        if (cudaMalloc((void**)&c->d_adj, adj_bytes) != cudaSuccess) return fail(SQZ_E_NOMEM);
        if (cudaMemset(c->d_adj, 0, adj_bytes) != cudaSuccess) return fail(SQZ_E_CUDA);
        TileParams q = tile_params(c);
        if (launch_tile_adjacency(q, c->d_adj, nullptr) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
          return fail(SQZ_E_CUDA);
      }
    }
    *out_ctx = c;
    return SQZ_OK;
  });
}

void squeeze_destroy(void* ctx) {
  if (!ctx) return;
  Ctx* c = static_cast<Ctx*>(ctx);
  free_device(c);
  delete c;
}

squeeze_status squeeze_geometry(const void* ctx, squeeze_geometry_t* out) {
  if (!ctx || !out) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  std::memset(out, 0, sizeof(*out));
  out->cells_total = c->V;
  out->omega_lo = c->sr.omega_lo;
  out->omega_hi = c->sr.omega_hi;
  out->state_bytes = c->state_bytes;
  out->n = c->n;
  out->compact_w = c->cw;
  out->compact_h = c->ch;
  out->r = c->r;
  out->tile_level = c->tt.g;
  out->tile_cells = c->tt.K;
  out->num_tiles = c->NT;
  out->chunk_tiles = kChunkTiles;
  out->remote_links = c->tt.E;
  out->max_degree = c->tt.max_degree;
  out->tile_bytes = c->Kp;
  out->packed_bytes = c->packed_bytes;
  out->chunk_words = c->Kw;
  out->packed_tiles = kPackTiles;
  out->heat_bytes = c->heat_bytes;
  out->heat_chunk_tiles = 4;
  out->heat_pairs = c->heat_P;
  out->byte_kernel = c->stream ? 1u : 0u;
  out->packed_ok = c->packed_grid > 0 ? 1u : 0u;
  out->heat_ok = c->heat_grid > 0 ? 1u : 0u;
  return SQZ_OK;
}

squeeze_status squeeze_shard_range(const void* ctx, uint32_t rank, uint64_t* lo, uint64_t* hi) {
  if (!ctx || !lo || !hi) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (rank >= c->nranks) return SQZ_E_CONFIG;
  ShardRange sr = shard_range(c->NT, c->tt.K, rank, c->nranks);
  *lo = sr.omega_lo;
  *hi = sr.omega_hi;
  return SQZ_OK;
}

squeeze_status squeeze_lambda_host(const void* ctx, uint64_t omega, uint32_t* x, uint32_t* y) {
  if (!ctx || !x || !y) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (omega >= c->V) return SQZ_E_OUT_OF_BOUNDS;
  lambda_level(c->full.view, omega, *x, *y);
  return SQZ_OK;
}

squeeze_status squeeze_nu_host(const void* ctx, uint64_t x, uint64_t y, uint64_t* omega) {
  if (!ctx || !omega) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (x >= c->n || y >= c->n) return SQZ_E_OUT_OF_BOUNDS;
  uint64_t om = nu_level(c->full.view, (int64_t)x, (int64_t)y);
  if (om == kNoneU64) return SQZ_E_HOLE;
  *omega = om;
  return SQZ_OK;
}

squeeze_status squeeze_map_lambda(const void* ctx, const uint64_t* d_omega, uint32_t* d_x, uint32_t* d_y,
                                  uint64_t count, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  if (count && (!d_omega || !d_x || !d_y)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_map_lambda(c->d_full.view, d_omega, d_x, d_y, count, (cudaStream_t)stream));
}

squeeze_status squeeze_map_nu(const void* ctx, const uint32_t* d_x, const uint32_t* d_y, uint64_t* d_omega,
                              uint64_t count, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  if (count && (!d_omega || !d_x || !d_y)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_map_nu(c->d_full.view, d_x, d_y, d_omega, count, (cudaStream_t)stream));
}

squeeze_status squeeze_map_nu_mma(const void* ctx, const uint32_t* d_x, const uint32_t* d_y, uint64_t* d_omega,
                                  uint64_t count, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  if (!c->d_mma_B) return SQZ_E_CONFIG;  // s^2 > 256 or k > 256: no u8 encoding
  if (count && (!d_omega || !d_x || !d_y)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  MmaNuParams q{};
  q.r = c->r;
  q.s = c->f.s;
  q.k = c->f.k;
  q.s_log2 = c->full.view.s_log2;
  q.n = c->n;
  q.hnu = c->d_mma_h;
  q.B = c->d_mma_B;
  return cu(launch_map_nu_mma(q, d_x, d_y, d_omega, count, (cudaStream_t)stream));
}

squeeze_status squeeze_seed(const void* ctx, uint8_t* d_state, uint64_t seed, uint64_t q, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_state);
  if (st != SQZ_OK) return st;
  if (q > (1ull << 32)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_seed(c->d_full.view, pad_layout(c), d_state, seed, q, (cudaStream_t)stream));
}

squeeze_status squeeze_step(void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st == SQZ_OK) st = check_state(c, d_next);
  if (st != SQZ_OK) return st;
  if (d_cur == d_next) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return do_step(c, d_cur, d_next, (cudaStream_t)stream);
}

squeeze_status squeeze_step_naive(void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st == SQZ_OK) st = check_state(c, d_next);
  if (st != SQZ_OK) return st;
  if (d_cur == d_next) return SQZ_E_CONFIG;
  if (c->nranks > 1 && !c->needs.empty() && c->d_recv == nullptr) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_step_naive(c->d_full.view, d_cur, d_next, c->rule.birth_mask, c->rule.survive_mask, halo_view(c),
                              (cudaStream_t)stream));
}

squeeze_status squeeze_run(void* ctx, uint8_t* d_a, uint8_t* d_b, uint64_t steps, int use_graph,
                           squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_a == d_b) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t pairs = steps / 2;
  if (use_graph && pairs > 0) {
    if (!(c->graph && c->graph_a == d_a && c->graph_b == d_b && c->graph_stream == s)) {
      if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
      }
      cudaStream_t cap;
      if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) return SQZ_E_CUDA;
      cudaGraph_t graph;
      if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaStreamDestroy(cap);
        return SQZ_E_CUDA;
      }
      squeeze_status s1 = do_step(c, d_a, d_b, cap);
      squeeze_status s2 = do_step(c, d_b, d_a, cap);
      cudaError_t ce = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      if (s1 != SQZ_OK || s2 != SQZ_OK || ce != cudaSuccess) return SQZ_E_CUDA;
      ce = cudaGraphInstantiate(&c->graph, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) return SQZ_E_CUDA;
      c->graph_a = d_a;
      c->graph_b = d_b;
      c->graph_stream = s;
    }
    for (uint64_t i = 0; i < pairs; ++i)
      if (cudaGraphLaunch(c->graph, s) != cudaSuccess) return SQZ_E_CUDA;
  } else {
    for (uint64_t i = 0; i < pairs; ++i) {
      if ((st = do_step(c, d_a, d_b, s)) != SQZ_OK) return st;
      if ((st = do_step(c, d_b, d_a, s)) != SQZ_OK) return st;
    }
  }
  if (steps & 1) return do_step(c, d_a, d_b, s);
  return SQZ_OK;
}

squeeze_status squeeze_run_host(void* ctx, uint8_t* h_state, uint8_t* d_a, uint8_t* d_b, uint64_t steps,
                                squeeze_stream_t stream) {
  if (!ctx || !h_state) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_a == d_b) return SQZ_E_CONFIG;  // before any transfer is enqueued
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(d_a, h_state, c->state_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) return SQZ_E_CUDA;
  if ((st = squeeze_run(ctx, d_a, d_b, steps, 0, stream)) != SQZ_OK) return st;
  const uint8_t* fin = (steps & 1) ? d_b : d_a;
  if (cudaMemcpyAsync(h_state, fin, c->state_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) return SQZ_E_CUDA;
  return cu(cudaStreamSynchronize(s));
}

squeeze_status squeeze_run_host_bits(void* ctx, uint32_t* h_packed, uint8_t* d_a, uint8_t* d_b, uint32_t* d_packed,
                                    uint64_t steps, squeeze_stream_t stream) {
  if (!ctx || !h_packed) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st == SQZ_OK) st = check_state(c, d_packed);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_a == d_b) return SQZ_E_CONFIG;  // before any transfer is enqueued
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // The state crosses PCIe at 1 bit per cell (the packed layout); the step runs on bytes.  The
  // transfers run on a second stream in segments of whole 128-tile packed chunks, so each
  // segment's unpack overlaps the next segment's H2D and each segment's D2H the next one's pack.
  const TileParams p = tile_params(c);
  const uint64_t ntiles = p.tile_hi - p.tile_lo, nch = (ntiles + kPackTiles - 1) / kPackTiles;
  const uint64_t per = nch ? (nch + 7) / 8 : 0, nseg = nch ? (nch + per - 1) / per : 1;  // no empty segments
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> ev(2 * nseg + 2, nullptr);
  auto cleanup = [&](squeeze_status r) {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
    return r;
  };
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return cleanup(SQZ_E_CUDA);
  for (cudaEvent_t& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return cleanup(SQZ_E_CUDA);
  auto seg = [&](uint64_t i, TileParams& q, uint64_t& poff, uint64_t& boff, uint64_t& pbytes) {
    const uint64_t c0 = i * per, c1 = std::min(nch, c0 + per);
    q = p;
    q.tile_lo = 0;
    q.tile_hi = std::min(ntiles, c1 * kPackTiles) - c0 * kPackTiles;
    poff = c0 * (uint64_t)c->Kw * 4;  // u32 words
    boff = c0 * kPackTiles * (uint64_t)c->Kp;
    pbytes = (c1 - c0) * (uint64_t)c->Kw * 16;
  };
  if (cudaEventRecord(ev[2 * nseg], s) != cudaSuccess || cudaStreamWaitEvent(cs, ev[2 * nseg], 0) != cudaSuccess)
    return cleanup(SQZ_E_CUDA);
  for (uint64_t i = 0; i < nseg && nch; ++i) {  // H2D (copy stream) -> unpack (stream), segment by segment
    TileParams q;
    uint64_t poff, boff, pbytes;
    seg(i, q, poff, boff, pbytes);
    if (cudaMemcpyAsync(d_packed + poff, h_packed + poff, pbytes, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaEventRecord(ev[i], cs) != cudaSuccess || cudaStreamWaitEvent(s, ev[i], 0) != cudaSuccess)
      return cleanup(SQZ_E_CUDA);
    if ((st = cu(launch_unpack(q, d_packed + poff, d_a + boff, s))) != SQZ_OK) return cleanup(st);
  }
  if ((st = squeeze_run(ctx, d_a, d_b, steps, 1, stream)) != SQZ_OK) return cleanup(st);
  const uint8_t* fin = (steps & 1) ? d_b : d_a;
  for (uint64_t i = 0; i < nseg && nch; ++i) {  // pack (stream) -> D2H (copy stream), segment by segment
    TileParams q;
    uint64_t poff, boff, pbytes;
    seg(i, q, poff, boff, pbytes);
    if ((st = cu(launch_pack(q, fin + boff, d_packed + poff, s))) != SQZ_OK) return cleanup(st);
    if (cudaEventRecord(ev[nseg + i], s) != cudaSuccess || cudaStreamWaitEvent(cs, ev[nseg + i], 0) != cudaSuccess ||
        cudaMemcpyAsync(h_packed + poff, d_packed + poff, pbytes, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      return cleanup(SQZ_E_CUDA);
  }
  if (cudaEventRecord(ev[2 * nseg + 1], cs) != cudaSuccess || cudaStreamWaitEvent(s, ev[2 * nseg + 1], 0) != cudaSuccess)
    return cleanup(SQZ_E_CUDA);
  return cleanup(cu(cudaStreamSynchronize(s)));
}

squeeze_status squeeze_run_host_packed(void* ctx, uint32_t* h_packed, uint32_t* d_a, uint32_t* d_b, uint64_t steps,
                                       squeeze_stream_t stream) {
  if (!ctx || !h_packed) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_a == d_b) return SQZ_E_CONFIG;  // before any transfer is enqueued
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(d_a, h_packed, c->packed_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) return SQZ_E_CUDA;
  if ((st = squeeze_run_packed(ctx, d_a, d_b, steps, stream)) != SQZ_OK) return st;
  const uint32_t* fin = (steps & 1) ? d_b : d_a;
  if (cudaMemcpyAsync(h_packed, fin, c->packed_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) return SQZ_E_CUDA;
  return cu(cudaStreamSynchronize(s));
}

squeeze_status squeeze_count_alive(const void* ctx, const uint8_t* d_state, uint64_t* d_out, squeeze_stream_t stream) {
  if (!ctx || !d_out) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_state);
  if (st != SQZ_OK) return st;
  DevGuard g(c->device);
  return cu(launch_count_alive(d_state, c->state_bytes, d_out, (cudaStream_t)stream));
}

squeeze_status squeeze_device_error(const void* ctx) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  DevGuard g(c->device);
  int flag = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return SQZ_E_CUDA;
  if (cudaMemcpy(&flag, c->d_err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return SQZ_E_CUDA;
  // read-and-reset: a miss is reported once, by the first call after the step that missed
  if (flag && cudaMemset(c->d_err, 0, sizeof(int)) != cudaSuccess) return SQZ_E_CUDA;
  return flag ? SQZ_E_HALO : SQZ_OK;
}

squeeze_status squeeze_halo_needs(const void* ctx, uint64_t* out, uint64_t cap, uint64_t* count) {
  if (!ctx || !count) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  *count = c->needs.size();
  if (out) std::memcpy(out, c->needs.data(), std::min<uint64_t>(cap, c->needs.size()) * sizeof(uint64_t));
  return SQZ_OK;
}

squeeze_status squeeze_halo_set_sends(void* ctx, const uint64_t* omegas, uint64_t count) {
  return guarded([&]() -> squeeze_status {
    if (!ctx || (count && !omegas)) return SQZ_E_CONFIG;
    Ctx* c = static_cast<Ctx*>(ctx);
    for (uint64_t i = 0; i < count; ++i)
      if (omegas[i] < c->sr.omega_lo || omegas[i] >= c->sr.omega_hi) return SQZ_E_CONFIG;
    c->sends.assign(omegas, omegas + count);
    if (c->device >= 0) {  // a peer plan indexes the old send list: drop it (re-plan after this call)
      DevGuard g(c->device);
      for (auto** q : {&c->d_peer_chunk_start, &c->d_peer_cell, &c->d_peer_of, &c->d_send_peer}) {
        cudaFree(*q);
        *q = nullptr;
      }
      for (auto** q : {&c->d_peer_pos, &c->d_send_pos}) {
        cudaFree(*q);
        *q = nullptr;
      }
      c->peer_parity = -1;
      if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
      }
    }
    c->send_offsets.resize(count);
    c->send_bits.resize(count);
    for (uint64_t i = 0; i < count; ++i) {  // tile-padded byte offsets / packed bits of the cells to send
      const uint64_t t = omegas[i] / c->tt.K, j = omegas[i] - t * c->tt.K, tl = t - c->sr.tile_lo;
      c->send_offsets[i] = tl * c->Kp + j;
      c->send_bits[i] = ((((tl / kPackTiles) * c->Kw + j) * 4 + (tl / 32) % 4) << 5) | (tl % 32);
    }
    if (c->device >= 0) {
      DevGuard g(c->device);
      cudaFree(c->d_sends);
      cudaFree(c->d_send_bits);
      c->d_sends = nullptr;
      c->d_send_bits = nullptr;
      squeeze_status st = upload(&c->d_sends, c->send_offsets.data(), c->send_offsets.size());
      if (st == SQZ_OK) st = upload(&c->d_send_bits, c->send_bits.data(), c->send_bits.size());
      return st;
    }
    return SQZ_OK;
  });
}

squeeze_status squeeze_halo_bind(void* ctx, uint8_t* d_send, const uint8_t* d_recv) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  if ((!c->sends.empty() && !d_send) || (!c->needs.empty() && !d_recv)) return SQZ_E_CONFIG;
  c->d_send = d_send;
  c->d_recv = d_recv;
  return SQZ_OK;
}

squeeze_status squeeze_halo_pack(const void* ctx, const uint8_t* d_cur, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st != SQZ_OK) return st;
  if (!c->sends.empty() && !c->d_send) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_halo_pack(d_cur, c->d_sends, c->sends.size(), c->d_send, (cudaStream_t)stream));
}

squeeze_status squeeze_ipc_handle(const void* d_ptr, uint8_t* handle) {
  if (!d_ptr || !handle) return SQZ_E_CONFIG;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)) != cudaSuccess) return SQZ_E_CUDA;
  std::memcpy(handle, &h, sizeof(h));
  return SQZ_OK;
}

squeeze_status squeeze_ipc_open(const uint8_t* handle, int device, void** d_ptr) {
  if (!handle || !d_ptr) return SQZ_E_CONFIG;
  DevGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cu(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

squeeze_status squeeze_ipc_close(void* d_ptr) { return d_ptr ? cu(cudaIpcCloseMemHandle(d_ptr)) : SQZ_OK; }

squeeze_status squeeze_ipc_alloc(uint64_t bytes, int device, void** d_ptr) {
  if (!d_ptr) return SQZ_E_CONFIG;
  DevGuard g(device);
  if (cudaMalloc(d_ptr, bytes ? bytes : 1) != cudaSuccess) return SQZ_E_NOMEM;
  return cu(cudaMemset(*d_ptr, 0, bytes ? bytes : 1));
}

squeeze_status squeeze_ipc_free(void* d_ptr) { return d_ptr ? cu(cudaFree(d_ptr)) : SQZ_OK; }

squeeze_status squeeze_halo_peer_push(const void* ctx, const uint8_t* d_cur, int parity, squeeze_stream_t stream) {
  if (!ctx || parity < 0 || parity > 1) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st != SQZ_OK) return st;
  if (c->sends.empty()) return SQZ_OK;
  if (!c->d_peer_recv[parity] || !c->d_peer_chunk_start || c->peer_slots[parity] != c->nranks) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_halo_peer_push(d_cur, c->d_sends, c->d_send_peer, c->d_send_pos, c->sends.size(),
                                  c->d_peer_recv[parity], (cudaStream_t)stream));
}

squeeze_status squeeze_halo_peer_plan(void* ctx, const uint32_t* send_peer, const uint64_t* send_pos) {
  return guarded([&]() -> squeeze_status {
    if (!ctx) return SQZ_E_CONFIG;
    Ctx* c = static_cast<Ctx*>(ctx);
    if (c->device < 0) return SQZ_E_NO_DEVICE;
    const uint64_t n = c->sends.size();
    if (n && (!send_peer || !send_pos)) return SQZ_E_CONFIG;
    // every destination is another rank of this context (peer slot = rank; the step kernel stores
    // through peer_recv[slot], so an out-of-range slot would write through a wild pointer)
    for (uint64_t i = 0; i < n; ++i)
      if (send_peer[i] >= c->nranks || send_peer[i] == c->rank) return SQZ_E_CONFIG;
    // CSR over the tile kernel's 32-tile chunks; cell = tile in chunk << 16 | j
    const uint64_t nch = (c->sr.tile_hi - c->sr.tile_lo + kChunkTiles - 1) / kChunkTiles;
    std::vector<uint32_t> start(nch + 1, 0), cell(n), of(n);
    std::vector<uint64_t> pos(n);
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t tl = c->sends[i] / c->tt.K - c->sr.tile_lo;
      start[tl / kChunkTiles + 1]++;
      order[i] = i;
    }
    for (uint64_t k = 0; k < nch; ++k) start[k + 1] += start[k];
    std::vector<uint32_t> fill(start.begin(), start.end() - 1);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t t = c->sends[i] / c->tt.K, tl = t - c->sr.tile_lo;
      const uint32_t e = fill[tl / kChunkTiles]++;
      cell[e] = (uint32_t)((tl % kChunkTiles) << 16 | (c->sends[i] - t * c->tt.K));
      of[e] = send_peer[i];
      pos[e] = send_pos[i];
    }
    DevGuard g(c->device);
    cudaFree(c->d_peer_chunk_start);
    cudaFree(c->d_peer_cell);
    cudaFree(c->d_peer_of);
    cudaFree(c->d_peer_pos);
    cudaFree(c->d_send_peer);
    cudaFree(c->d_send_pos);
    c->d_send_peer = nullptr;
    c->d_send_pos = nullptr;
    c->d_peer_chunk_start = nullptr;
    c->d_peer_cell = c->d_peer_of = nullptr;
    c->d_peer_pos = nullptr;
    squeeze_status st = upload(&c->d_peer_chunk_start, start.data(), start.size());
    if (st == SQZ_OK) st = upload(&c->d_peer_cell, cell.data(), cell.size());
    if (st == SQZ_OK) st = upload(&c->d_peer_of, of.data(), of.size());
    if (st == SQZ_OK) st = upload(&c->d_peer_pos, pos.data(), pos.size());
    if (st == SQZ_OK) st = upload(&c->d_send_peer, send_peer, n);
    if (st == SQZ_OK) st = upload(&c->d_send_pos, send_pos, n);
    return st;
  });
}

squeeze_status squeeze_halo_peer_bind(void* ctx, uint32_t parity, uint32_t npeers, void* const* peer_recv) {
  if (!ctx || parity > 1 || (npeers && !peer_recv)) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (c->device < 0) return SQZ_E_NO_DEVICE;
  // one pointer per rank (slot = rank); the own slot is never stored through
  if (npeers != 0 && npeers != c->nranks) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  cudaFree(c->d_peer_recv[parity]);
  c->d_peer_recv[parity] = nullptr;
  c->peer_slots[parity] = npeers;
  if (npeers == 0) return SQZ_OK;
  return upload(&c->d_peer_recv[parity], reinterpret_cast<uint8_t* const*>(peer_recv), npeers);
}

squeeze_status squeeze_halo_peer_select(void* ctx, int parity) {
  if (!ctx || parity > 1 || parity < -1) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (parity >= 0 && (!c->d_peer_chunk_start || (!c->d_peer_recv[parity] && !c->sends.empty())))
    return SQZ_E_CONFIG;
  if (parity >= 0 && !c->sends.empty() && c->peer_slots[parity] != c->nranks) return SQZ_E_CONFIG;
  c->peer_parity = parity;
  if (c->graph) {  // a captured run would replay the old parameters
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  return SQZ_OK;
}

squeeze_status squeeze_halo_pack_packed(const void* ctx, const uint32_t* d_cur, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st != SQZ_OK) return st;
  if (!c->sends.empty() && !c->d_send) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_halo_pack_packed(d_cur, c->d_send_bits, c->sends.size(), c->d_send, (cudaStream_t)stream));
}

squeeze_status squeeze_pack(const void* ctx, const uint8_t* d_state, uint32_t* d_packed, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_state);
  if (st == SQZ_OK) st = check_state(c, d_packed);
  if (st != SQZ_OK) return st;
  DevGuard g(c->device);
  return cu(launch_pack(tile_params(c), d_state, d_packed, (cudaStream_t)stream));
}

squeeze_status squeeze_unpack(const void* ctx, const uint32_t* d_packed, uint8_t* d_state, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_state);
  if (st == SQZ_OK) st = check_state(c, d_packed);
  if (st != SQZ_OK) return st;
  DevGuard g(c->device);
  return cu(launch_unpack(tile_params(c), d_packed, d_state, (cudaStream_t)stream));
}

squeeze_status squeeze_seed_packed(const void* ctx, uint32_t* d_packed, uint64_t seed, uint64_t q,
                                   squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_packed);
  if (st != SQZ_OK) return st;
  if (q > (1ull << 32)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_seed_packed(tile_params(c), c->d_full.view, d_packed, seed, q, (cudaStream_t)stream));
}

squeeze_status squeeze_step_packed(void* ctx, const uint32_t* d_cur, uint32_t* d_next, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st == SQZ_OK) st = check_state(c, d_next);
  if (st != SQZ_OK) return st;
  if ((const void*)d_cur == (const void*)d_next) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return do_step_packed(c, d_cur, d_next, (cudaStream_t)stream);
}

squeeze_status squeeze_run_packed(void* ctx, uint32_t* d_a, uint32_t* d_b, uint64_t steps, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st != SQZ_OK) return st;
  if (d_a == d_b || c->nranks > 1) return SQZ_E_CONFIG;  // sharded: step + halo exchange per step
  DevGuard g(c->device);
  for (uint64_t i = 0; i < steps; ++i) {
    st = (i & 1) ? do_step_packed(c, d_b, d_a, (cudaStream_t)stream) : do_step_packed(c, d_a, d_b, (cudaStream_t)stream);
    if (st != SQZ_OK) return st;
  }
  return SQZ_OK;
}

squeeze_status squeeze_count_alive_packed(const void* ctx, const uint32_t* d_packed, uint64_t* d_out,
                                          squeeze_stream_t stream) {
  if (!ctx || !d_out) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_packed);
  if (st != SQZ_OK) return st;
  DevGuard g(c->device);
  return cu(launch_count_packed(d_packed, c->packed_bytes / 4, d_out, (cudaStream_t)stream));
}

squeeze_status squeeze_heat_seed(const void* ctx, float* d_u, uint64_t seed, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_u);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_heat_seed(c->d_full.view, tile_params(c), d_u, seed, (cudaStream_t)stream));
}

squeeze_status squeeze_heat_step(void* ctx, const float* d_cur, float* d_next, float alpha, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st == SQZ_OK) st = check_state(c, d_next);
  if (st != SQZ_OK) return st;
  if (d_cur == d_next || !(alpha == alpha)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return do_heat_step(c, d_cur, d_next, alpha, (cudaStream_t)stream);
}

squeeze_status squeeze_heat_run(void* ctx, float* d_a, float* d_b, uint64_t steps, float alpha,
                                squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  Ctx* c = static_cast<Ctx*>(ctx);
  squeeze_status st = check_state(c, d_a);
  if (st == SQZ_OK) st = check_state(c, d_b);
  if (st != SQZ_OK) return st;
  if (d_a == d_b || !(alpha == alpha)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  for (uint64_t i = 0; i < steps && st == SQZ_OK; ++i)
    st = (i & 1) ? do_heat_step(c, d_b, d_a, alpha, (cudaStream_t)stream)
                 : do_heat_step(c, d_a, d_b, alpha, (cudaStream_t)stream);
  return st;
}

squeeze_status squeeze_heat_sum(const void* ctx, const float* d_u, double* d_out, squeeze_stream_t stream) {
  if (!ctx || !d_out) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_u);
  if (st != SQZ_OK) return st;
  DevGuard g(c->device);
  return cu(launch_heat_sum(d_u, c->heat_bytes / 4, d_out, (cudaStream_t)stream));
}

squeeze_status squeeze_lambda_engine_step(const void* ctx, const uint8_t* d_cur_grid, uint8_t* d_next_grid,
                                          squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur_grid);
  if (st == SQZ_OK) st = check_state(c, d_next_grid);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_cur_grid == d_next_grid || c->n > (1ull << 20)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_lambda_engine(c->d_full.view, d_cur_grid, d_next_grid, c->rule.birth_mask, c->rule.survive_mask,
                                 (cudaStream_t)stream));
}

squeeze_status squeeze_block_bytes(const void* ctx, uint32_t rho, uint64_t* bytes) {
  if (!ctx || !bytes) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  const int m = block_m(c, rho);
  if (m < 0) return SQZ_E_INVALID_LEVEL;
  uint64_t nb;
  if (!checked_pow(c->f.k, c->r - (uint32_t)m, 1ull << 56, nb)) return SQZ_E_OVERFLOW;
  *bytes = nb * rho * rho;
  return SQZ_OK;
}

squeeze_status squeeze_block_seed(void* ctx, uint32_t rho, uint8_t* d_blocks, uint64_t seed, uint64_t q,
                                  squeeze_stream_t stream) {
  return guarded([&]() -> squeeze_status {
    if (!ctx) return SQZ_E_CONFIG;
    Ctx* c = static_cast<Ctx*>(ctx);
    squeeze_status st = check_state(c, d_blocks);
    if (st != SQZ_OK) return st;
    if (c->nranks > 1 || q > (1ull << 32)) return SQZ_E_CONFIG;
    DevGuard g(c->device);
    BlockLevel* bl;
    if ((st = block_level(c, rho, &bl)) != SQZ_OK) return st;
    return cu(launch_block_seed(bl->dev.view, rho, bl->d_micro, d_blocks, seed, q, (cudaStream_t)stream));
  });
}

squeeze_status squeeze_block_step(void* ctx, uint32_t rho, const uint8_t* d_cur, uint8_t* d_next,
                                  squeeze_stream_t stream) {
  return guarded([&]() -> squeeze_status {
    if (!ctx) return SQZ_E_CONFIG;
    Ctx* c = static_cast<Ctx*>(ctx);
    squeeze_status st = check_state(c, d_cur);
    if (st == SQZ_OK) st = check_state(c, d_next);
    if (st != SQZ_OK) return st;
    if (c->nranks > 1 || d_cur == d_next) return SQZ_E_CONFIG;
    DevGuard g(c->device);
    BlockLevel* bl;
    if ((st = block_level(c, rho, &bl)) != SQZ_OK) return st;
    return cu(launch_block_step(bl->dev.view, rho, bl->d_micro, c->rule.birth_mask, c->rule.survive_mask, d_cur,
                                d_next, (cudaStream_t)stream));
  });
}

squeeze_status squeeze_bb_bytes(const void* ctx, uint64_t* bytes) {
  if (!ctx || !bytes) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (c->n > (1ull << 20)) return SQZ_E_OVERFLOW;
  *bytes = c->n * c->n;
  return SQZ_OK;
}

squeeze_status squeeze_bb_seed(const void* ctx, uint8_t* d_grid, uint64_t seed, uint64_t q, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_grid);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || q > (1ull << 32) || c->n > (1ull << 20)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_bb_seed(c->d_full.view, d_grid, seed, q, (cudaStream_t)stream));
}

squeeze_status squeeze_bb_step(const void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_cur);
  if (st == SQZ_OK) st = check_state(c, d_next);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1 || d_cur == d_next || c->n > (1ull << 20)) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_bb_step(d_cur, d_next, c->n, c->rule.birth_mask, c->rule.survive_mask, (cudaStream_t)stream));
}

squeeze_status squeeze_bb_to_compact(const void* ctx, const uint8_t* d_grid, uint8_t* d_state,
                                     squeeze_stream_t stream) {
  if (!ctx) return SQZ_E_CONFIG;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  squeeze_status st = check_state(c, d_grid);
  if (st == SQZ_OK) st = check_state(c, d_state);
  if (st != SQZ_OK) return st;
  if (c->nranks > 1) return SQZ_E_CONFIG;
  DevGuard g(c->device);
  return cu(launch_bb_to_compact(c->d_full.view, pad_layout(c), d_grid, d_state, (cudaStream_t)stream));
}

}  // extern "C"
