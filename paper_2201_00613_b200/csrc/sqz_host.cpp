// sqz_host.cpp — host-side planner of the Squeeze hot path.  See sqz_host.h.
#include "sqz_host.h"

#include <algorithm>
#include <map>
#include <thread>

#include "../../include/squeeze.h"

namespace sqz {

int make_spec(uint32_t k, uint32_t s, const uint8_t* tau, Spec& out) {
  // S:29-33 invariants: s >= 2, 1 <= k <= s^2, τ injective with components in [0, s-1]
  // (replicas "can be translated, but cannot rotate neither overlap").
  if (s < 2 || s > 256 || k < 1 || (uint64_t)k > (uint64_t)s * s || tau == nullptr) return SQZ_E_INVALID_SPEC;
  out.k = k;
  out.s = s;
  out.tau.assign(tau, tau + 2 * k);
  out.hnu.assign((size_t)s * s, -1);
  for (uint32_t b = 0; b < k; ++b) {
    uint32_t tx = tau[2 * b], ty = tau[2 * b + 1];
    if (tx >= s || ty >= s) return SQZ_E_INVALID_SPEC;
    int& slot = out.hnu[(size_t)ty * s + tx];
    if (slot != -1) return SQZ_E_INVALID_SPEC;
    slot = (int)b;  // H_ν inverts H_λ on replica quadrants
  }
  return SQZ_OK;
}

bool builtin_spec(const std::string& name, uint32_t& k, uint32_t& s, std::vector<uint8_t>& tau) {
  // Sierpinski triangle τ(0)=(0,0), τ(1)=(0,1), τ(2)=(1,1): P:224.  The other layouts
  // are drawn only in the paper's figures (reading D11).
  static const std::map<std::string, std::pair<std::pair<uint32_t, uint32_t>, std::vector<uint8_t>>> table = {
      {"sierpinski-triangle", {{3, 2}, {0, 0, 0, 1, 1, 1}}},
      {"sierpinski-carpet", {{8, 3}, {0, 0, 1, 0, 2, 0, 0, 1, 2, 1, 0, 2, 1, 2, 2, 2}}},
      {"vicsek", {{5, 3}, {0, 0, 2, 0, 1, 1, 0, 2, 2, 2}}},
      {"empty-bottles", {{7, 3}, {1, 0, 0, 1, 1, 1, 2, 1, 0, 2, 1, 2, 2, 2}}},
      {"full-square", {{4, 2}, {0, 0, 1, 0, 0, 1, 1, 1}}},
  };
  auto it = table.find(name);
  if (it == table.end()) return false;
  k = it->second.first.first;
  s = it->second.first.second;
  tau = it->second.second;
  return true;
}

FastDiv64 make_fastdiv(uint64_t d) {
  FastDiv64 f{};
  f.d = d;
  if (d <= 1) {
    f.one = 1;
    return f;
  }
  uint32_t l = 63 - (uint32_t)__builtin_clzll(d);
  if ((d & (d - 1)) == 0) {  // power of two: q = (n >> 1) >> (l - 1)
    f.magic = 0;
    f.shift = l - 1;
    return f;
  }
  unsigned __int128 num = (unsigned __int128)1 << (64 + l);
  uint64_t m = (uint64_t)(num / d);
  uint64_t rem = (uint64_t)(num % d);
  m += m;  // 65-bit magic, low 64 bits (wraps by design)
  uint64_t twice = rem + rem;
  if (twice >= d || twice < rem) m += 1;
  f.magic = m + 1;
  f.shift = l;
  return f;
}

bool checked_pow(uint64_t base, uint32_t e, uint64_t limit, uint64_t& out) {
  unsigned __int128 v = 1;
  for (uint32_t i = 0; i < e; ++i) {
    v *= base;
    if (v > limit) return false;
  }
  out = (uint64_t)v;
  return true;
}

static uint64_t ipow(uint64_t b, uint32_t e) {
  uint64_t v = 1;
  for (uint32_t i = 0; i < e; ++i) v *= b;
  return v;
}

// λ partial of a digits (Σ τ(digit_i) s^i), packed x | y << 16.
static uint32_t lam_partial(const Spec& f, uint64_t d, uint32_t a) {
  uint32_t x = 0, y = 0, sc = 1;
  for (uint32_t i = 0; i < a; ++i) {
    uint32_t b = (uint32_t)(d % f.k);
    d /= f.k;
    x += f.tau[2 * b] * sc;
    y += f.tau[2 * b + 1] * sc;
    sc *= f.s;
  }
  return x | (y << 16);
}

// ν partial over b base-s digits of (xd, yd): Σ H_ν[θ_i] k^i or HOLE.
static uint32_t nu_partial(const Spec& f, uint32_t xd, uint32_t yd, uint32_t b) {
  uint64_t om = 0, sc = 1;
  for (uint32_t i = 0; i < b; ++i) {
    uint32_t tx = xd % f.s, ty = yd % f.s;
    xd /= f.s;
    yd /= f.s;
    int h = f.hnu[(size_t)ty * f.s + tx];
    if (h < 0) return kHoleU32;
    om += (uint64_t)h * sc;
    sc *= f.k;
  }
  return (uint32_t)om;
}

void build_level_maps(const Spec& f, uint32_t L, HostLevelMaps& out) {
  LevelMaps& m = out.view;
  m = LevelMaps{};
  m.levels = L;
  m.k = f.k;
  m.s = f.s;
  // λ group size: k^a <= 4096 and s^a < 65536 (partial coordinates packed in 16 bits)
  uint32_t a = 1;
  while (a < 16 && ipow(f.k, a + 1) <= 4096 && ipow(f.s, a + 1) < 65536) ++a;
  // ν group size: (s^b)^2 <= 4096 entries and k^b < 2^31 (partial Ω, HOLE sentinel)
  uint32_t b = 1;
  while (b < 16 && ipow(f.s, 2 * (b + 1)) <= 4096 && ipow(f.k, b + 1) < (1ull << 31)) ++b;
  m.a = a;
  m.a_full = L / a;
  m.a_tail = L % a;
  m.b = b;
  m.b_full = L / b;
  m.b_tail = L % b;
  m.sa = (uint32_t)ipow(f.s, a);
  m.sb = (uint32_t)ipow(f.s, b);
  m.sb_tail = (uint32_t)ipow(f.s, m.b_tail);
  m.s_log2 = ((f.s & (f.s - 1)) == 0) ? (uint32_t)__builtin_ctz(f.s) : 0;
  m.n = ipow(f.s, L);
  m.cells = ipow(f.k, L);
  m.kb = ipow(f.k, b);
  m.div_ka = make_fastdiv(ipow(f.k, a));
  m.div_sb = make_fastdiv(m.sb);
  uint64_t ka = ipow(f.k, a);
  out.lam_full.resize(ka);
  for (uint64_t d = 0; d < ka; ++d) out.lam_full[d] = lam_partial(f, d, a);
  uint64_t kt = ipow(f.k, m.a_tail);
  out.lam_tail.resize(kt);
  for (uint64_t d = 0; d < kt; ++d) out.lam_tail[d] = lam_partial(f, d, m.a_tail);
  out.nu_full.resize((size_t)m.sb * m.sb);
  for (uint32_t yd = 0; yd < m.sb; ++yd)
    for (uint32_t xd = 0; xd < m.sb; ++xd) out.nu_full[(size_t)yd * m.sb + xd] = nu_partial(f, xd, yd, b);
  out.nu_tail.resize((size_t)m.sb_tail * m.sb_tail);
  for (uint32_t yd = 0; yd < m.sb_tail; ++yd)
    for (uint32_t xd = 0; xd < m.sb_tail; ++xd)
      out.nu_tail[(size_t)yd * m.sb_tail + xd] = nu_partial(f, xd, yd, m.b_tail);
  m.n_lam_full = (uint32_t)out.lam_full.size();
  m.n_lam_tail = (uint32_t)out.lam_tail.size();
  m.n_nu_full = (uint32_t)out.nu_full.size();
  m.n_nu_tail = (uint32_t)out.nu_tail.size();
  m.lam_full = out.lam_full.data();
  m.lam_tail = out.lam_tail.data();
  m.nu_full = out.nu_full.data();
  m.nu_tail = out.nu_tail.data();
}

uint32_t auto_tile_level(const Spec& f, uint32_t r, uint64_t max_cells) {
  uint32_t g = 0;
  while (g < r && ipow(f.k, g + 1) <= max_cells && ipow(f.s, 2 * (g + 1)) <= (1ull << 20)) ++g;
  return g;
}

int build_tile_tables(const Spec& f, uint32_t g, TileTables& t) {
  t = TileTables{};
  t.g = g;
  uint64_t K, h;
  if (!checked_pow(f.k, g, 1u << 15, K) || !checked_pow(f.s, g, 1u << 12, h)) return SQZ_E_INVALID_LEVEL;
  t.K = K;
  t.h = h;
  // local λ_g and its inverse on the h x h tile embedding
  t.local_x.resize(K);
  t.local_y.resize(K);
  std::vector<int32_t> inv((size_t)h * h, -1);
  for (uint64_t j = 0; j < K; ++j) {
    uint64_t d = j, x = 0, y = 0, sc = 1;
    for (uint32_t i = 0; i < g; ++i) {
      uint32_t b = (uint32_t)(d % f.k);
      d /= f.k;
      x += f.tau[2 * b] * sc;
      y += f.tau[2 * b + 1] * sc;
      sc *= f.s;
    }
    t.local_x[j] = (uint32_t)x;
    t.local_y[j] = (uint32_t)y;
    inv[(size_t)y * h + x] = (int32_t)j;
  }
  // neighbour entries: local j' (< K) or remote link K + e; remote links are shared by
  // every tile because each level-g sub-fractal is a translated copy (NBB class)
  std::vector<std::vector<uint32_t>> entries(K);
  std::map<uint64_t, uint32_t> remote_index;
  int dir_of[9];
  for (int i = 0; i < 9; ++i) dir_of[i] = -1;
  for (uint64_t j = 0; j < K; ++j) {
    for (int i = 0; i < 8; ++i) {
      int64_t xx = (int64_t)t.local_x[j] + moore_dx(i);
      int64_t yy = (int64_t)t.local_y[j] + moore_dy(i);
      int dx = xx < 0 ? -1 : (xx >= (int64_t)h ? 1 : 0);
      int dy = yy < 0 ? -1 : (yy >= (int64_t)h ? 1 : 0);
      uint64_t lx = (uint64_t)(xx - dx * (int64_t)h), ly = (uint64_t)(yy - dy * (int64_t)h);
      int32_t jj = inv[(size_t)ly * h + lx];
      if (jj < 0) continue;  // a hole of the level-g fractal: never a member neighbour
      if (dx == 0 && dy == 0) {
        entries[j].push_back((uint32_t)jj);
      } else {
        int key = (dx + 1) + 3 * (dy + 1);
        if (dir_of[key] < 0) {
          dir_of[key] = (int)t.ndirs;
          t.dir_dx[t.ndirs] = dx;
          t.dir_dy[t.ndirs] = dy;
          ++t.ndirs;
        }
        // one remote word per distinct (direction, neighbour-tile cell): several own cells
        // that touch the same outside cell share it
        const uint64_t rkey = (uint64_t)dir_of[key] * K + (uint64_t)jj;
        auto found = remote_index.find(rkey);
        uint32_t e;
        if (found == remote_index.end()) {
          e = (uint32_t)t.link_j2.size();
          remote_index.emplace(rkey, e);
          t.link_j.push_back((uint32_t)j);
          t.link_j2.push_back((uint32_t)jj);
          t.link_dir.push_back((uint8_t)dir_of[key]);
        } else {
          e = found->second;
        }
        entries[j].push_back((uint32_t)(K + e));
      }
    }
  }
  t.E = (uint32_t)t.link_j.size();
  t.zero_slot = (uint32_t)(K + t.E);
  if (t.zero_slot > 0xFFFFu) return SQZ_E_INVALID_LEVEL;
  // sort links by direction (stable) so each direction's links are contiguous
  std::vector<uint32_t> order(t.E), where(t.E);
  for (uint32_t e = 0; e < t.E; ++e) order[e] = e;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return t.link_dir[a] < t.link_dir[b]; });
  std::vector<uint32_t> lj(t.E), lj2(t.E);
  std::vector<uint8_t> ld(t.E);
  for (uint32_t e = 0; e < t.E; ++e) {
    lj[e] = t.link_j[order[e]];
    lj2[e] = t.link_j2[order[e]];
    ld[e] = t.link_dir[order[e]];
    where[order[e]] = e;
  }
  t.link_j.swap(lj);
  t.link_j2.swap(lj2);
  t.link_dir.swap(ld);
  t.dir_start.assign(t.ndirs + 1, 0);
  for (uint32_t e = 0; e < t.E; ++e) t.dir_start[t.link_dir[e] + 1]++;
  for (uint32_t d = 0; d < t.ndirs; ++d) t.dir_start[d + 1] += t.dir_start[d];
  t.nbr.assign(K * 8, (uint16_t)t.zero_slot);
  for (uint64_t j = 0; j < K; ++j) {
    t.max_degree = std::max<uint32_t>(t.max_degree, (uint32_t)entries[j].size());
    for (size_t e = 0; e < entries[j].size(); ++e) {
      uint32_t v = entries[j][e];
      if (v >= K) v = (uint32_t)(K + where[v - K]);
      t.nbr[j * 8 + e] = (uint16_t)v;
    }
  }
  return SQZ_OK;
}

namespace {
// wavefronts of one slot across the lanes of a quarter: the largest number of DISTINCT words
// that share a 16-byte bank group (word mod 8); equal words are one broadcast
int slot_wavefronts(const uint16_t* w, int n) {
  uint16_t seen[8];
  int ns = 0, cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, best = 0;
  for (int l = 0; l < n; ++l) {
    bool dup = false;
    for (int s = 0; s < ns; ++s) dup |= seen[s] == w[l];
    if (dup) continue;
    seen[ns++] = w[l];
    best = std::max(best, ++cnt[w[l] & 7]);
  }
  return best;
}
}  // namespace

void optimize_slot_order(std::vector<uint16_t>& rows, uint64_t K, int D) {
  for (uint64_t q0 = 0; q0 < K; q0 += 8) {
    const int n = (int)std::min<uint64_t>(8, K - q0);
    auto cost = [&]() {
      int c = 0;
      for (int k = 0; k < D; ++k) {
        uint16_t w[8];
        for (int l = 0; l < n; ++l) w[l] = rows[(q0 + l) * 8 + k];
        c += slot_wavefronts(w, n);
      }
      return c;
    };
    int best = cost();
    for (int pass = 0; pass < 8; ++pass) {
      const int before = best;
      for (int l = 0; l < n; ++l) {
        uint16_t* r = &rows[(q0 + l) * 8];
        if (D <= 5) {  // every permutation of this lane's D slots
          int idx[5] = {0, 1, 2, 3, 4};
          uint16_t orig[5], keep[5];
          for (int k = 0; k < D; ++k) orig[k] = keep[k] = r[k];
          do {
            for (int k = 0; k < D; ++k) r[k] = orig[idx[k]];
            const int c = cost();
            if (c < best) {
              best = c;
              for (int k = 0; k < D; ++k) keep[k] = r[k];
            }
          } while (std::next_permutation(idx, idx + D));
          for (int k = 0; k < D; ++k) r[k] = keep[k];
        } else {  // pairwise swaps
          for (int a = 0; a < D; ++a)
            for (int b = a + 1; b < D; ++b) {
              std::swap(r[a], r[b]);
              const int c = cost();
              if (c < best) best = c;
              else std::swap(r[a], r[b]);
            }
        }
      }
      if (best == before) break;
    }
  }
}

ShardRange shard_range(uint64_t num_tiles, uint64_t K, uint32_t rank, uint32_t nranks) {
  uint64_t nchunks = (num_tiles + kChunkTiles - 1) / kChunkTiles;
  uint64_t c_lo = (uint64_t)((unsigned __int128)nchunks * rank / nranks);
  uint64_t c_hi = (uint64_t)((unsigned __int128)nchunks * (rank + 1) / nranks);
  ShardRange sr;
  sr.tile_lo = std::min<uint64_t>(c_lo * kChunkTiles, num_tiles);
  sr.tile_hi = std::min<uint64_t>(c_hi * kChunkTiles, num_tiles);
  sr.omega_lo = sr.tile_lo * K;
  sr.omega_hi = sr.tile_hi * K;
  return sr;
}

void halo_needs(const TileTables& t, const LevelMaps& coarse, const ShardRange& sr, std::vector<uint64_t>& out,
                unsigned threads) {
  out.clear();
  uint64_t ntiles = sr.tile_hi - sr.tile_lo;
  if (ntiles == 0 || t.E == 0) return;
  threads = std::max(1u, std::min<unsigned>(threads, (unsigned)std::min<uint64_t>(ntiles / 4096 + 1, 256)));
  std::vector<std::vector<uint64_t>> parts(threads);
  auto work = [&](unsigned w) {
    uint64_t a = sr.tile_lo + ntiles * w / threads, b = sr.tile_lo + ntiles * (w + 1) / threads;
    std::vector<uint64_t>& mine = parts[w];
    for (uint64_t tile = a; tile < b; ++tile) {
      uint32_t X, Y;
      lambda_level(coarse, tile, X, Y);
      for (uint32_t d = 0; d < t.ndirs; ++d) {
        uint64_t nt = nu_level(coarse, (int64_t)X + t.dir_dx[d], (int64_t)Y + t.dir_dy[d]);
        if (nt == kNoneU64 || (nt >= sr.tile_lo && nt < sr.tile_hi)) continue;
        for (uint32_t e = 0; e < t.E; ++e)
          if (t.link_dir[e] == d) mine.push_back(nt * t.K + t.link_j2[e]);
      }
    }
    std::sort(mine.begin(), mine.end());
    mine.erase(std::unique(mine.begin(), mine.end()), mine.end());
  };
  std::vector<std::thread> pool;
  for (unsigned w = 1; w < threads; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& th : pool) th.join();
  for (auto& p : parts) out.insert(out.end(), p.begin(), p.end());
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

}  // namespace sqz
