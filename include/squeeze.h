/*
 * squeeze.h — C ABI of the B200-native Squeeze hot path (arXiv 2201.00613).
 *
 * One automaton step on the COMPACT form of an NBB fractal (§3, §4):
 * for every compact cell Ω, λ(Ω) gives its expanded (x, y), the 8
 * Moore neighbours are tested for membership ("the holes were skipped"),
 * ν maps each member neighbour back to a compact index, the states
 * are gathered, the rule applied and the result written to a second buffer
 * ("at most one execution of λ(ω) map and ℓ executions of ν(ω)").
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper used here):
 *  - Ω is the compact index Σ_{μ=1..r} β_μ k^{μ-1} (reading D2): digit μ-1 of Ω in
 *    base k is the replica id at level μ.  A state buffer holds one uint8 per
 *    cell (0 dead / 1 alive, reading D10) in Ω order, TILE-PADDED: Ω = t·K + j
 *    (K = k^g cells per level-g tile) lives at byte offset
 *    (t - t_lo)·Kp + j, Kp = tile_bytes = K rounded up to 32, plus 16 when that is an
 *    even multiple of 16, so every tile starts on a 16-byte boundary, a run of tiles
 *    moves with one TMA bulk copy, and 128-bit lane accesses are bank-conflict-free.
 *    The Kp - K padding bytes of each tile are zero (3.2% of the buffer for K = 729).
 *    INPUT CONTRACT of the stepping kernels: every cell byte is 0 or 1 and every padding
 *    byte is 0 (squeeze_seed, squeeze_step, squeeze_unpack and the binding's from_cells
 *    keep it; the kernels pack bytes with shifted adds).  A buffer breaking it yields
 *    unspecified cell values, never an out-of-bounds access.
 *  - (x, y) is the expanded coordinate, origin upper-left, y downward.
 *  - Level μ of x/y has weight s^{μ-1}; axis parity per reading D1.
 *
 * Ownership: every device pointer passed in is CALLER-owned (torch allocations in
 * the Python binding), contiguous and 16-byte aligned; state buffers must be at
 * least `state_bytes` long (squeeze_geometry).  A sharded context's local buffer
 * holds the tiles [t_lo, t_hi) of Ω in [omega_lo, omega_hi).  The context owns its
 * lookup tables, tile tables and halo index arrays, freed by squeeze_destroy.
 * All device calls are asynchronous and stream-ordered on the given stream; a
 * context is not thread-safe.  No C++ exception crosses this boundary: every
 * entry point returns a squeeze_status (negative on error).
 */
#ifndef SQUEEZE_H_
#define SQUEEZE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* squeeze_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  SQZ_OK = 0,
  SQZ_E_INVALID_SPEC = -1,   /* fractal violates S:29-33 (s>=2, 1<=k<=s^2, τ injective, τ in [0,s-1]^2) */
  SQZ_E_OVERFLOW = -2,       /* s^r > 2^32 (coordinates) or k^r >= 2^62 (Ω) */
  SQZ_E_OUT_OF_BOUNDS = -3,  /* scalar map argument outside the compact range / n x n embedding */
  SQZ_E_HOLE = -4,           /* scalar ν of a non-member (D5) */
  SQZ_E_INVALID_LEVEL = -5,  /* level or tile level out of range */
  SQZ_E_CONFIG = -6,         /* NULL/misaligned pointer, bad shard, missing halo binding, buffer too small */
  SQZ_E_CUDA = -7,           /* a CUDA runtime call failed (asynchronous faults surface on a later call) */
  SQZ_E_NO_DEVICE = -8,      /* device entry point called on a host-only context (device = -1) */
  SQZ_E_NOMEM = -9,          /* host or device allocation failed */
  SQZ_E_HALO = -10           /* a kernel needed a neighbour outside the shard that the halo plan lacks */
} squeeze_status;

/* An NBB fractal F(n, k, s): k replicas per level, scale s per level, and the
 * replica offset table τ = H_λ: tau[2b] = τ_x(b), tau[2b+1] = τ_y(b). */
typedef struct {
  uint32_t k;
  uint32_t s;
  const uint8_t* tau; /* 2k bytes, host memory, copied by squeeze_init */
} squeeze_fractal;

/* Life-like rule (reading D6): a dead cell with c member neighbours is born iff bit c
 * of birth_mask is set; a live one survives iff bit c of survive_mask is set (c <= 8).
 * Conway's B3/S23 is {1<<3, (1<<2)|(1<<3)}. */
typedef struct {
  uint16_t birth_mask;
  uint16_t survive_mask;
} squeeze_rule;

/* Data-parallel sharding of Ω by contiguous, chunk-aligned ranges.
 * nranks = 1 is the unsharded case.  Shard ranges are computed identically by every
 * rank from (fractal, r, nranks). */
typedef struct {
  uint32_t rank;
  uint32_t nranks;
} squeeze_shard;

/* Tuning knobs; zero-initialise for defaults. */
typedef struct {
  uint32_t tile_level;    /* g: level of the compact tile (K = k^g cells); 0 = auto (largest K <= 1024) */
  uint32_t block_threads; /* threads per CTA of the tile kernel; 0 = auto */
  uint32_t ctas_per_sm;   /* persistent CTAs per SM; 0 = auto (occupancy) */
} squeeze_options;

typedef struct {
  uint64_t cells_total;  /* V = k^r */
  uint64_t omega_lo;     /* first Ω owned by this shard */
  uint64_t omega_hi;     /* one past the last Ω owned */
  uint64_t state_bytes;  /* required bytes of a state buffer: local tiles x tile_bytes */
  uint64_t n;            /* expanded side s^r */
  uint64_t compact_w;    /* k^⌊r/2⌋ (D1) */
  uint64_t compact_h;    /* k^⌈r/2⌉ */
  uint32_t r;            /* level */
  uint32_t tile_level;   /* g actually used */
  uint64_t tile_cells;   /* K = k^g */
  uint64_t num_tiles;    /* k^(r-g) in the whole fractal */
  uint32_t chunk_tiles;  /* tiles per CTA work unit (32: one bit-slice lane per tile) */
  uint32_t remote_links; /* tile-boundary neighbour links per tile (table size) */
  uint32_t max_degree;   /* largest neighbour-slot count of any cell of a tile (<= 8) */
  uint32_t tile_bytes;   /* Kp: bytes per tile in a state buffer (K rounded up to 32, odd multiple of 16) */
  uint64_t packed_bytes; /* bytes of a PACKED state buffer (squeeze_*_packed) */
  uint32_t chunk_words;  /* Kw: 128-bit words per chunk in the packed layout (K rounded up to 4) */
  uint32_t packed_tiles; /* tiles per chunk of the packed layout (128) */
  uint64_t heat_bytes;   /* bytes of a HEAT field buffer (squeeze_heat_*) */
  uint32_t heat_chunk_tiles; /* tiles per chunk of the heat layout (4: one float4 word per cell) */
  uint32_t heat_pairs;   /* remote (own cell, neighbour) pairs per tile of the heat kernel */
  uint32_t byte_kernel;  /* squeeze_step's kernel: 0 = chunk-staged (k_step_tile), 1 = streaming
                          * large-tile step (k_step_stream, when a 32-tile chunk does not fit shared
                          * memory twice); both compute the same step on the same layout */
  uint32_t packed_ok;    /* 1 if the packed step fits at this tile level (else its calls return
                          * SQZ_E_INVALID_LEVEL): the 128-tile chunk fits shared memory twice and its
                          * boundary links need at most 64 link work items (a tile with very long
                          * edges, e.g. a hollow square with s=12 at tile level 2, does not) */
  uint32_t heat_ok;      /* 1 if the heat step fits at this tile level (likewise) */
} squeeze_geometry_t;

const char* squeeze_strerror(squeeze_status st);
const char* squeeze_version(void);

/* Look up a built-in fractal by name ("sierpinski-triangle", "sierpinski-carpet",
 * "vicsek", "empty-bottles", "full-square").  `tau_out` receives 2k bytes (cap >= 2k).
 * Returns SQZ_E_INVALID_SPEC for an unknown name. */
squeeze_status squeeze_builtin_fractal(const char* name, uint32_t* k, uint32_t* s, uint8_t* tau_out,
                                       uint32_t cap);

/* Create a context for fractal `f` at level `r` (r = log_s n).  `rule` NULL means
 * B3/S23; `shard` NULL means unsharded; `opts` NULL means defaults.  device >= 0 binds
 * the context to that CUDA device and uploads its tables (sets that device current);
 * device = -1 creates a HOST-ONLY context: geometry, scalar maps and halo planning work,
 * device entry points return SQZ_E_NO_DEVICE.  Validates the spec and that
 * s^r <= 2^32 and k^r < 2^62.  For nranks > 1 the halo plan (squeeze_halo_needs) is
 * built here on the host. */
squeeze_status squeeze_init(void** out_ctx, const squeeze_fractal* f, uint32_t r, const squeeze_rule* rule,
                            const squeeze_shard* shard, const squeeze_options* opts, int device);
void squeeze_destroy(void* ctx);

squeeze_status squeeze_geometry(const void* ctx, squeeze_geometry_t* out);

/* Shard range of any rank under this context's (fractal, r, nranks). */
squeeze_status squeeze_shard_range(const void* ctx, uint32_t rank, uint64_t* lo, uint64_t* hi);

/* ---- scalar host twins of the maps (tests and tooling; no device needed) ---- */
/* λ(Ω): Ω in [0, k^r) -> expanded (x, y); SQZ_E_OUT_OF_BOUNDS otherwise. */
squeeze_status squeeze_lambda_host(const void* ctx, uint64_t omega, uint32_t* x, uint32_t* y);
/* ν(x, y): member -> Ω; SQZ_E_HOLE on a hole, SQZ_E_OUT_OF_BOUNDS outside n x n. */
squeeze_status squeeze_nu_host(const void* ctx, uint64_t x, uint64_t y, uint64_t* omega);

/* ---- batched device maps; `count` elements; device pointers; async on `stream` ---- */
/* d_x[i], d_y[i] = λ(d_omega[i]); Ω >= k^r yields x = y = UINT32_MAX. */
squeeze_status squeeze_map_lambda(const void* ctx, const uint64_t* d_omega, uint32_t* d_x, uint32_t* d_y,
                                  uint64_t count, squeeze_stream_t stream);
/* d_omega[i] = ν(d_x[i], d_y[i]); holes and out-of-range coordinates yield UINT64_MAX. */
squeeze_status squeeze_map_nu(const void* ctx, const uint32_t* d_x, const uint32_t* d_y, uint64_t* d_omega,
                              uint64_t count, squeeze_stream_t stream);
/* ν as an exact integer tensor-core product (SURVEY §8f NEXT-3 ablation of P:296-332):
 * Ω = Σ_b (A·B)[c][b] 256^b with A[c][μ] = H_ν[θ_μ(c)] (u8) and B[μ][b] = byte b of k^(μ-1),
 * one mma.sync m16n8k32 u8 per 16 coordinates.  Same contract and output as squeeze_map_nu;
 * SQZ_E_CONFIG when s^2 > 256 or k > 256 (no u8 encoding).  Not on the hot path: bench.py
 * times it beside the LUT map. */
squeeze_status squeeze_map_nu_mma(const void* ctx, const uint32_t* d_x, const uint32_t* d_y, uint64_t* d_omega,
                                  uint64_t count, squeeze_stream_t stream);

/* ---- automaton ---- */
/* Initial state (reading D9): cell Ω alive iff (mix(((X<<32)|Y) ^ mix(seed)) >> 32) < q at
 * (X, Y) = λ(Ω), mix = splitmix64 finaliser; q = round(density * 2^32) in [0, 2^32].
 * Writes state_bytes bytes (padding zeroed). */
squeeze_status squeeze_seed(const void* ctx, uint8_t* d_state, uint64_t seed, uint64_t q,
                            squeeze_stream_t stream);
/* One synchronous step d_next = F(d_cur) with the tile-amortised bit-sliced kernel
 * (DESIGN.md §5).  d_cur and d_next must not alias.  A sharded context reads
 * out-of-shard neighbours from the halo receive buffer bound by squeeze_halo_bind,
 * which the caller must have filled for d_cur's generation. */
squeeze_status squeeze_step(void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream);
/* The same step computed literally per cell (one λ and eight membership tests + ν per
 * cell): the paper's per-thread formulation, kept as a comparison engine. */
squeeze_status squeeze_step_naive(void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream);
/* `steps` steps ping-ponging d_a -> d_b -> d_a ...; the final state is in d_b if steps is
 * odd, else d_a.  Unsharded contexts only (SQZ_E_CONFIG otherwise).  use_graph != 0
 * captures the two-step ping-pong once into a CUDA graph and replays it. */
squeeze_status squeeze_run(void* ctx, uint8_t* d_a, uint8_t* d_b, uint64_t steps, int use_graph,
                           squeeze_stream_t stream);
/* End to end from HOST memory: copies h_state (the tile-padded state, state_bytes long, ideally
 * pinned) to d_a, runs `steps` steps, copies the final state back into h_state, and synchronises
 * `stream`.  d_a, d_b are caller-owned device scratch buffers.  Unsharded contexts only:
 * SQZ_E_CONFIG (before any copy is enqueued) for a sharded context or aliased d_a == d_b.  The
 * library cannot see the host buffer's length: the caller guarantees state_bytes. */
squeeze_status squeeze_run_host(void* ctx, uint8_t* h_state, uint8_t* d_a, uint8_t* d_b, uint64_t steps,
                                squeeze_stream_t stream);
/* End to end from host memory with the state crossing PCIe at 1 BIT per cell: h_packed holds the
 * state in the packed layout (packed_bytes, see the packed section below; squeeze_pack/_unpack
 * convert on the device), d_packed is a caller-owned device buffer of packed_bytes.  H2D of
 * h_packed, unpack into d_a, `steps` byte-state steps (the CUDA-graph ping-pong of squeeze_run),
 * pack of the final state, D2H into h_packed, synchronise.  The state is binary, so this moves 8x
 * fewer bytes over PCIe than squeeze_run_host for the same result.  The transfers run on an
 * internal copy stream in up to 8 segments of whole 128-tile packed chunks, ordered after prior
 * work on `stream`: each segment's unpack overlaps the next one's H2D, each segment's D2H the next
 * one's pack; the call returns after everything completed.  Unsharded contexts only (SQZ_E_CONFIG
 * before any copy otherwise). */
squeeze_status squeeze_run_host_bits(void* ctx, uint32_t* h_packed, uint8_t* d_a, uint8_t* d_b, uint32_t* d_packed,
                                    uint64_t steps, squeeze_stream_t stream);
/* *d_out (device uint64) = number of alive cells of this shard. */
squeeze_status squeeze_count_alive(const void* ctx, const uint8_t* d_state, uint64_t* d_out,
                                   squeeze_stream_t stream);
/* Reads AND CLEARS the device-side error flag (synchronises the device): SQZ_E_HALO once for
 * every run of steps in which a kernel missed a halo cell, then SQZ_OK again. */
squeeze_status squeeze_device_error(const void* ctx);

/* ---- halo exchange plan for sharded contexts (data moved by the caller, e.g. NCCL) ---- */
/* Sorted, unique global Ω outside this shard that some in-shard cell has as a member
 * neighbour.  Writes min(cap, total) entries, *count = total.  out may be NULL. */
squeeze_status squeeze_halo_needs(const void* ctx, uint64_t* out, uint64_t cap, uint64_t* count);
/* Ω (inside this shard) whose states this shard must send each step, in send-buffer order. */
squeeze_status squeeze_halo_set_sends(void* ctx, const uint64_t* omegas, uint64_t count);
/* Caller-owned device buffers: d_send receives `send count` bytes from squeeze_halo_pack;
 * d_recv holds one byte per squeeze_halo_needs entry, in that order. */
squeeze_status squeeze_halo_bind(void* ctx, uint8_t* d_send, const uint8_t* d_recv);
/* d_send[i] = state of cell sends[i] in d_cur. */
squeeze_status squeeze_halo_pack(const void* ctx, const uint8_t* d_cur, squeeze_stream_t stream);

/* ---- peer-memory halo: the step kernel stores the halo itself (fused transport) ----
 * Instead of squeeze_halo_pack + a collective, squeeze_step's epilogue writes each send cell of
 * its OUTPUT straight into the receiving rank's buffer over NVLink (CUDA IPC mappings), so the
 * next step's halo is in place when the step ends; the caller only orders steps across ranks
 * (e.g. a barrier after each step) and alternates two receive buffers by step parity.
 * squeeze_ipc_handle / _open / _close: cudaIpc{Get,Open,Close}MemHandle (64-byte handles).
 * squeeze_halo_peer_plan: destination of every send (squeeze_halo_set_sends order): peer slot
 *   send_peer[i] (the destination RANK: < nranks and != this rank, else SQZ_E_CONFIG) and byte
 *   position send_pos[i] in that peer's receive buffer (the caller's plan guarantees it is below
 *   the receiver's squeeze_halo_needs count).  squeeze_halo_set_sends drops an existing peer plan.
 * squeeze_halo_peer_bind: device pointers (IPC-opened) of the peers' receive buffers for one
 *   parity, indexed by peer slot: npeers must be 0 (unbind) or nranks (SQZ_E_CONFIG otherwise).  squeeze_halo_peer_select: parity the next squeeze_step writes
 *   (-1 = off, the default).  Byte state only (squeeze_step). */
squeeze_status squeeze_ipc_handle(const void* d_ptr, uint8_t* handle);
squeeze_status squeeze_ipc_open(const uint8_t* handle, int device, void** d_ptr);
squeeze_status squeeze_ipc_close(void* d_ptr);
/* Receive buffers for the peer halo: plain cudaMalloc'd, zeroed (an IPC handle names a whole
 * allocation, so these are not sub-allocations of a caching allocator). */
squeeze_status squeeze_ipc_alloc(uint64_t bytes, int device, void** d_ptr);
squeeze_status squeeze_ipc_free(void* d_ptr);
/* The halo of d_cur written into the peers' receive buffers of `parity` (the first step's halo;
 * afterwards squeeze_step's epilogue writes it). */
squeeze_status squeeze_halo_peer_push(const void* ctx, const uint8_t* d_cur, int parity, squeeze_stream_t stream);
squeeze_status squeeze_halo_peer_plan(void* ctx, const uint32_t* send_peer, const uint64_t* send_pos);
squeeze_status squeeze_halo_peer_bind(void* ctx, uint32_t parity, uint32_t npeers, void* const* peer_recv);
squeeze_status squeeze_halo_peer_select(void* ctx, int parity);

/* ---- bit-sliced PACKED state (1 bit per cell) ----
 * Layout: the shard's tiles are grouped in chunks of packed_tiles = 128 consecutive tiles;
 * chunk c holds Kw 128-bit words (packed_bytes = chunks x Kw x 16); 32-bit lane q (0..3) of
 * word j, bit i = cell j of tile 128c + 32q + i of the shard, i.e. the u32 at index
 * (c x Kw + j) x 4 + q (j < K; padding words and bits of tiles past the shard end are zero).
 * It is the form the step computes on, so a packed step moves 0.25 B per cell instead of 2 B.
 * Sharded contexts: squeeze_step_packed reads out-of-shard neighbours from the bound halo receive
 * buffer (fill it as for squeeze_step, packing with squeeze_halo_pack_packed); squeeze_run_packed
 * is unsharded only (SQZ_E_CONFIG otherwise).  Buffers: 16-byte aligned device memory. */
squeeze_status squeeze_pack(const void* ctx, const uint8_t* d_state, uint32_t* d_packed, squeeze_stream_t stream);
squeeze_status squeeze_unpack(const void* ctx, const uint32_t* d_packed, uint8_t* d_state, squeeze_stream_t stream);
/* d_send[i] = state of cell sends[i] in a packed buffer (the packed twin of squeeze_halo_pack). */
squeeze_status squeeze_halo_pack_packed(const void* ctx, const uint32_t* d_cur, squeeze_stream_t stream);
/* D9 initial state written directly in the packed layout (same cells as squeeze_seed). */
squeeze_status squeeze_seed_packed(const void* ctx, uint32_t* d_packed, uint64_t seed, uint64_t q,
                                   squeeze_stream_t stream);
/* One synchronous step on packed buffers (d_cur, d_next must not alias). */
squeeze_status squeeze_step_packed(void* ctx, const uint32_t* d_cur, uint32_t* d_next, squeeze_stream_t stream);
/* `steps` packed steps ping-ponging d_a / d_b (final state in d_b if steps is odd). */
squeeze_status squeeze_run_packed(void* ctx, uint32_t* d_a, uint32_t* d_b, uint64_t steps, squeeze_stream_t stream);
/* End to end from host memory on the packed state (unsharded): H2D of h_packed (packed_bytes,
 * ideally pinned), `steps` packed steps, D2H of the final state into h_packed, synchronised. */
squeeze_status squeeze_run_host_packed(void* ctx, uint32_t* h_packed, uint32_t* d_a, uint32_t* d_b, uint64_t steps,
                                       squeeze_stream_t stream);
/* *d_out (device uint64) = number of alive cells in a packed buffer. */
squeeze_status squeeze_count_alive_packed(const void* ctx, const uint32_t* d_packed, uint64_t* d_out,
                                          squeeze_stream_t stream);

/* ---- second workload: heat diffusion on the compact fractal ----
 * Squeeze serves "PDE solvers, cellular-automata, spin-model simulations ... as they rely
 * on accessing neighboring cells".  One explicit step of the graph heat equation (D16):
 *     u'(Ω) = u(Ω) + α Σ_{n ∈ N(Ω)} (u(n) − u(Ω)),  N(Ω) = member Moore neighbours,
 * i.e. an insulated boundary; α·max_degree <= 1 keeps it a convex combination (stable).
 * Layout: float32 in chunks of heat_chunk_tiles = 4 consecutive tiles; chunk c holds K float4
 * words, word j = cell j of tiles 4c..4c+3, i.e. the float at index (c x K + j) x 4 + (t mod 4)
 * for local tile t (lanes of tiles past the shard end are 0); heat_bytes per buffer; 16-byte
 * aligned caller-owned device memory.  Unsharded contexts only
 * (SQZ_E_CONFIG otherwise); d_cur and d_next must not alias. */
/* Initial field: u(Ω) = (mix(((X<<32)|Y) ^ mix(seed)) >> 40) x 2^-24 at (X, Y) = λ(Ω). */
squeeze_status squeeze_heat_seed(const void* ctx, float* d_u, uint64_t seed, squeeze_stream_t stream);
squeeze_status squeeze_heat_step(void* ctx, const float* d_cur, float* d_next, float alpha, squeeze_stream_t stream);
/* `steps` steps ping-ponging d_a / d_b (final field in d_b if steps is odd). */
squeeze_status squeeze_heat_run(void* ctx, float* d_a, float* d_b, uint64_t steps, float alpha,
                                squeeze_stream_t stream);
/* *d_out (device double) = Σ u over the buffer (conserved by the step up to rounding). */
squeeze_status squeeze_heat_sum(const void* ctx, const float* d_u, double* d_out, squeeze_stream_t stream);

/* ---- the paper's comparison engines ---- */
/* λ(ω) engine ("compact grid and expanded fractal"): one thread per compact cell computes
 * λ(Ω) and updates that cell of an EXPANDED grid in the BB layout (squeeze_bb_*; 2 = hole). */
squeeze_status squeeze_lambda_engine_step(const void* ctx, const uint8_t* d_cur_grid, uint8_t* d_next_grid,
                                          squeeze_stream_t stream);
/* Block-level Squeeze with rho = s^m (m <= level, rho <= 32): k^(r-m) blocks, block b
 * holding the rho x rho expanded micro-embedding of its level-m sub-fractal at expanded origin
 * λ_{r-m}(b)·rho; byte (b·rho + y)·rho + x; 0 dead, 1 alive, 2 hole.  Unsharded contexts only. */
squeeze_status squeeze_block_bytes(const void* ctx, uint32_t rho, uint64_t* bytes);
squeeze_status squeeze_block_seed(void* ctx, uint32_t rho, uint8_t* d_blocks, uint64_t seed, uint64_t q,
                                  squeeze_stream_t stream);
squeeze_status squeeze_block_step(void* ctx, uint32_t rho, const uint8_t* d_cur, uint8_t* d_next,
                                  squeeze_stream_t stream);

/* ---- expanded bounding-box baseline (the paper's "BB" engine) ---- */
/* n x n uint8 grid, row-major [y][x]: 0 dead, 1 alive, 2 hole (never changes).  Unsharded only. */
squeeze_status squeeze_bb_bytes(const void* ctx, uint64_t* bytes);
squeeze_status squeeze_bb_seed(const void* ctx, uint8_t* d_grid, uint64_t seed, uint64_t q, squeeze_stream_t stream);
squeeze_status squeeze_bb_step(const void* ctx, const uint8_t* d_cur, uint8_t* d_next, squeeze_stream_t stream);
/* state of cell Ω in d_state = d_grid[λ(Ω)] — transports a BB grid to the compact layout. */
squeeze_status squeeze_bb_to_compact(const void* ctx, const uint8_t* d_grid, uint8_t* d_state,
                                     squeeze_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SQUEEZE_H_ */
