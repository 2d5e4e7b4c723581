// sqz_common.h — data structures shared by the host planner and the CUDA kernels of
// the Squeeze hot path.  Header-only pieces here compile for host and device.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SQZ_HD __host__ __device__ __forceinline__
#else
#define SQZ_HD inline
#endif

namespace sqz {

constexpr uint32_t kHoleU32 = 0xFFFFFFFFu;
constexpr uint64_t kNoneU64 = ~0ull;
constexpr int kChunkTiles = 32;  // one bit-slice lane per tile
constexpr uint32_t kPackTiles = 128;  // tiles per chunk of the packed layout (a 128-bit word per cell)

// ---------------------------------------------------------------------------
// Exact unsigned 64-bit division by a runtime-constant divisor, by multiply-high
// (the round-up "branch-free" method: q = (hi(m·n) + ((n - hi(m·n)) >> 1)) >> sh).
// Correct for every 64-bit n and every divisor d >= 1 (d = 1 handled by `one`).
struct FastDiv64 {
  uint64_t d;
  uint64_t magic;
  uint32_t shift;
  uint32_t one;  // d == 1
};

SQZ_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

SQZ_HD uint64_t fdiv(const FastDiv64& f, uint64_t n) {
  if (f.one) return n;
  uint64_t q = umulhi64(f.magic, n);
  uint64_t t = ((n - q) >> 1) + q;
  return t >> f.shift;
}

// ---------------------------------------------------------------------------
// Multi-digit lookup tables of one map at one level L:
//  λ: digits of Ω (base k) are consumed `a` at a time; lam_full[d] packs the
//     partial expanded offset Σ_{i<a} τ(digit_i) s^i as (x | y << 16).  The last
//     group has `a_tail` = L mod a digits and uses lam_tail (no padded digit may
//     contribute τ(0), which is non-zero for some fractals).
//  ν: base-s digits of x and y are consumed `b` at a time; nu_full[ybits*sb + xbits]
//     is the partial Ω Σ_{i<b} H_ν[θ_i] k^i, or kHoleU32 if some quadrant is a hole.
struct LevelMaps {
  uint32_t levels;     // L
  uint32_t k, s;
  uint32_t a, a_full, a_tail;  // λ digits per lookup, # full groups, tail digits
  uint32_t b, b_full, b_tail;  // ν digits per lookup, # full groups, tail digits
  uint32_t sa;                 // s^a
  uint32_t sb;                 // s^b
  uint32_t sb_tail;            // s^b_tail
  uint32_t s_log2;             // log2 s if s is a power of two, else 0
  uint64_t n;                  // s^L
  uint64_t cells;              // k^L
  uint64_t kb;                 // k^b
  FastDiv64 div_ka;            // division by k^a
  FastDiv64 div_sb;            // division by s^b
  uint32_t n_lam_full, n_lam_tail, n_nu_full, n_nu_tail;  // table lengths
  const uint32_t* lam_full;
  const uint32_t* lam_tail;
  const uint32_t* nu_full;
  const uint32_t* nu_tail;
};

// λ_L(Ω) -> (x, y); Ω < k^L assumed.
SQZ_HD void lambda_level(const LevelMaps& m, uint64_t omega, uint32_t& x, uint32_t& y) {
  uint64_t X = 0, Y = 0, scale = 1;
  for (uint32_t i = 0; i < m.a_full; ++i) {
    uint64_t q = fdiv(m.div_ka, omega);
    uint32_t d = (uint32_t)(omega - q * m.div_ka.d);
    omega = q;
    uint32_t p = m.lam_full[d];
    X += (uint64_t)(p & 0xFFFFu) * scale;
    Y += (uint64_t)(p >> 16) * scale;
    scale *= m.sa;
  }
  if (m.a_tail) {
    uint32_t p = m.lam_tail[(uint32_t)omega];
    X += (uint64_t)(p & 0xFFFFu) * scale;
    Y += (uint64_t)(p >> 16) * scale;
  }
  x = (uint32_t)X;
  y = (uint32_t)Y;
}

// ν_L(x, y) -> Ω or kNoneU64 (hole or outside [0, s^L)^2).  Signed inputs allow the
// Moore offsets of edge cells.
SQZ_HD uint64_t nu_level(const LevelMaps& m, int64_t sx, int64_t sy) {
  if (sx < 0 || sy < 0 || (uint64_t)sx >= m.n || (uint64_t)sy >= m.n) return kNoneU64;
  uint64_t x = (uint64_t)sx, y = (uint64_t)sy;
  uint64_t om = 0, scale = 1;
  for (uint32_t i = 0; i < m.b_full; ++i) {
    uint32_t xd, yd;
    if (m.s_log2) {
      xd = (uint32_t)(x & (m.sb - 1));
      yd = (uint32_t)(y & (m.sb - 1));
      x >>= m.s_log2 * m.b;
      y >>= m.s_log2 * m.b;
    } else {
      uint64_t qx = fdiv(m.div_sb, x), qy = fdiv(m.div_sb, y);
      xd = (uint32_t)(x - qx * m.sb);
      yd = (uint32_t)(y - qy * m.sb);
      x = qx;
      y = qy;
    }
    uint32_t p = m.nu_full[yd * m.sb + xd];
    if (p == kHoleU32) return kNoneU64;
    om += (uint64_t)p * scale;
    scale *= m.kb;
  }
  if (m.b_tail) {
    uint32_t p = m.nu_tail[(uint32_t)y * m.sb_tail + (uint32_t)x];
    if (p == kHoleU32) return kNoneU64;
    om += (uint64_t)p * scale;
  }
  return om;
}

// Moore offsets in a fixed order (row-major over the 3x3 stencil minus the centre).
SQZ_HD int moore_dx(int i) { return (i == 0 || i == 3 || i == 5) ? -1 : ((i == 1 || i == 6) ? 0 : 1); }
SQZ_HD int moore_dy(int i) { return i < 3 ? -1 : (i < 5 ? 0 : 1); }

}  // namespace sqz
