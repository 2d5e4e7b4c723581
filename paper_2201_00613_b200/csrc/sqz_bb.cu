// sqz_bb.cu — the expanded bounding-box (BB) engine of the paper's comparison ("BB"), the
// baseline of the compact-vs-expanded speedup (BASELINE configs[1], S = T_BB / T_compact).
//
// The BB state is the n x n expanded grid, one byte per cell: 0 dead, 1 alive, 2 hole (reading D8),
// so a step moves 2 B per EXPANDED cell and the kernel is HBM-bound.  To be an honest baseline it
// runs at the byte roofline: lane = a 32-cell strip of a row, the strip's cells bit-sliced into an
// alive plane and a hole plane (bit i = cell x0 + i), horizontal neighbours by shifts plus one
// shuffle per side, a warp walks down a band of rows keeping three rows of planes in registers
// (each row is read once), and the 8-neighbour count is a carry-save adder tree on whole words.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sqz_bits.cuh"

namespace sqz {

constexpr uint32_t kBBRows = 64;  // rows per warp band (two extra halo rows per band: +3% reads)

// 4 bytes in {0, 1} -> 4 bits, byte b -> bit b (the partial products of 0x01020408 never collide)
__device__ __forceinline__ uint32_t nib4(uint32_t w) { return (w * 0x01020408u) >> 24; }
// 4 bits -> 4 bytes in {0, 1}
__device__ __forceinline__ uint32_t unnib4(uint32_t b) { return (b * 0x00204081u) & 0x01010101u; }

struct RowRaw {
  uint4 lo, hi;
  uint32_t edge;  // lane 0: the byte left of the warp's segment; lane 31: the byte right of it
};

struct RowPlanes {
  uint32_t alive, hole, left, right;  // left/right: the alive plane moved by one cell (bit i = cell x0+i-1 / x0+i+1)
};

__device__ __forceinline__ RowRaw bb_load(const uint8_t* __restrict__ grid, uint32_t n, int64_t y, uint32_t x0,
                                         bool active, int lane) {
  RowRaw r;
  r.lo = make_uint4(0u, 0u, 0u, 0u);
  r.hi = r.lo;
  r.edge = 0;
  if (y < 0 || y >= (int64_t)n) return r;
  const uint8_t* row = grid + (uint64_t)y * n;
  if (active) {
    r.lo = __ldg(reinterpret_cast<const uint4*>(row + x0));
    r.hi = __ldg(reinterpret_cast<const uint4*>(row + x0 + 16));
    if (lane == 0 && x0 > 0) r.edge = __ldg(row + x0 - 1);
    if (lane == 31 && x0 + 32 < n) r.edge = __ldg(row + x0 + 32);
  }
  return r;
}

__device__ __forceinline__ RowPlanes bb_planes(const RowRaw& r, int lane) {
  const uint32_t w[8] = {r.lo.x, r.lo.y, r.lo.z, r.lo.w, r.hi.x, r.hi.y, r.hi.z, r.hi.w};
  RowPlanes p;
  p.alive = 0;
  p.hole = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    p.alive |= nib4(w[k] & 0x01010101u) << (4 * k);         // byte 1 -> alive (2 = hole has bit 0 clear)
    p.hole |= nib4((w[k] >> 1) & 0x01010101u) << (4 * k);  // byte 2 -> hole
  }
  const uint32_t edge_alive = r.edge == 1u ? 1u : 0u;
  uint32_t from_left = __shfl_up_sync(0xFFFFFFFFu, p.alive, 1) >> 31;   // cell x0 - 1
  uint32_t from_right = __shfl_down_sync(0xFFFFFFFFu, p.alive, 1) & 1u;  // cell x0 + 32
  if (lane == 0) from_left = edge_alive;
  if (lane == 31) from_right = edge_alive;
  p.left = (p.alive << 1) | from_left;
  p.right = (p.alive >> 1) | (from_right << 31);
  return p;
}

template <bool CONWAY>
__global__ void __launch_bounds__(256) k_bb_step_bits(const uint8_t* __restrict__ cur, uint8_t* __restrict__ next,
                                                      uint32_t n, uint32_t birth, uint32_t survive) {
  const int lane = threadIdx.x & 31;
  const uint32_t segs = (n + 1023) / 1024;  // 1024-cell row segments (one per warp)
  const uint32_t bands = (n + kBBRows - 1) / kBBRows;
  const uint32_t task = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (task >= segs * bands) return;
  const uint32_t band = task / segs, seg = task - band * segs;
  const uint32_t x0 = (seg * 32 + (uint32_t)lane) * 32;
  const bool active = x0 < n;
  const int64_t y0 = (int64_t)band * kBBRows;
  const int64_t y1 = min((int64_t)n, y0 + (int64_t)kBBRows);
  RowPlanes up = bb_planes(bb_load(cur, n, y0 - 1, x0, active, lane), lane);
  RowPlanes mid = bb_planes(bb_load(cur, n, y0, x0, active, lane), lane);
  RowRaw ahead = bb_load(cur, n, y0 + 1, x0, active, lane);
  for (int64_t y = y0; y < y1; ++y) {
    const RowPlanes dn = bb_planes(ahead, lane);
    ahead = bb_load(cur, n, y + 2, x0, active, lane);  // one row of loads in flight ahead of the compute
    // carry-save count of the 8 neighbour planes
    const uint32_t sa = up.left ^ up.alive ^ up.right, ka = maj3(up.left, up.alive, up.right);
    const uint32_t sb = dn.left ^ dn.alive ^ dn.right, kb = maj3(dn.left, dn.alive, dn.right);
    const uint32_t sc = sa ^ sb ^ mid.left, kc = maj3(sa, sb, mid.left);
    const uint32_t c0 = sc ^ mid.right;
    const uint32_t kd = sc & mid.right;
    const uint32_t se = ka ^ kb ^ kc, ke = maj3(ka, kb, kc);
    const uint32_t c1 = se ^ kd;
    const uint32_t kf = se & kd;
    const uint32_t c2 = ke ^ kf, c3 = ke & kf;
    const uint32_t alive = mid.alive;
    uint32_t nw;
    if (CONWAY) nw = c1 & ~c2 & ~c3 & (c0 | alive);  // B3/S23
    else nw = (alive & rule_bits(survive, c0, c1, c2, c3)) | (~alive & rule_bits(birth, c0, c1, c2, c3));
    nw &= ~mid.hole;  // holes stay 2, never alive
    if (active) {
      uint32_t o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = unnib4((nw >> (4 * k)) & 0xFu) | (unnib4((mid.hole >> (4 * k)) & 0xFu) << 1);
      uint8_t* row = next + (uint64_t)y * n + x0;
      *reinterpret_cast<uint4*>(row) = make_uint4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<uint4*>(row + 16) = make_uint4(o[4], o[5], o[6], o[7]);
    }
    up = mid;
    mid = dn;
  }
}

// n % 32 == 0 (every power-of-two n >= 32); other n take the per-cell kernel of sqz_kernels.cu.
bool bb_bits_ok(uint64_t n) { return n >= 32 && n % 32 == 0 && n <= (1ull << 31); }

cudaError_t launch_bb_step_bits(const uint8_t* cur, uint8_t* next, uint64_t n, uint32_t birth, uint32_t survive,
                                cudaStream_t st) {
  const uint64_t warps = ((n + 1023) / 1024) * ((n + kBBRows - 1) / kBBRows);
  const uint64_t blocks = (warps + 7) / 8;
  const bool conway = birth == (1u << 3) && survive == ((1u << 2) | (1u << 3));
  if (conway) k_bb_step_bits<true><<<(unsigned)blocks, 256, 0, st>>>(cur, next, (uint32_t)n, birth, survive);
  else k_bb_step_bits<false><<<(unsigned)blocks, 256, 0, st>>>(cur, next, (uint32_t)n, birth, survive);
  return cudaGetLastError();
}

}  // namespace sqz
