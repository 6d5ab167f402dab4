// Host planner: the stream-K decomposition and mapping of LeanTiles (§4.3, Alg. 2 §4-18).
//
// P:412  "Each CTAs range of LeanTile iterations is mapped contiguously into the batch size
//         -> heads -> context length linearization, crossing the head and query boundary as
//         it may ... each attention output tile is consolidated by the CTA that performed that
//         output's first LeanTile (called as a host block)."
// P:432  ragged: "mapped contiguously in a Heads -> TotalContextLength linearization".
// Eq. 2 / Alg2§6-9: I = sum_u C_n(u), equal contiguous ranges per CTA.
//
// Integer work only; tests check it bit-exactly against the oracle's independent
// enumeration (tests/test_planner.py).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "la_internal.h"

namespace la {

int64_t Problem::kv_rows() const {
  if (layout == LA_KV_BHSD) return int64_t(batch) * heads_kv * max_ctx;
  if (layout == LA_KV_PAGED) return num_pages * heads_kv * page_size;
  int64_t total = 0;
  for (int32_t n : ctx_lens) total += n;
  return int64_t(heads_kv) * total;
}

void build_units(const Problem& p, int tile_n, std::vector<DevUnit>& units, int64_t& total_iters) {
  units.clear();
  units.reserve(size_t(p.batch) * p.heads_kv);
  std::vector<int64_t> cu(p.batch + 1, 0), cq(p.batch + 1, 0);  // cu_seqlens, query rows
  for (int b = 0; b < p.batch; ++b) {
    cu[b + 1] = cu[b] + p.ctx_lens[b];
    cq[b + 1] = cq[b] + int64_t(p.heads_q) * p.q_lens[b];
  }
  int64_t it = 0;
  auto add = [&](int b, int h) {
    // query tiles m = 0 .. C_m - 1 of T_m rows over the g * N_b rows (Alg2§4 C_m), each a
    // unit that streams the whole KV of (b, h) -- innermost, so tiles of one KV run together
    const int nq = p.q_lens[b], rows = p.group * nq;
    for (int r0 = 0; r0 < rows; r0 += p.tile_rows) {
      DevUnit u{};
      u.len = p.ctx_lens[b];
      if (p.layout == LA_KV_BHSD)
        u.row0 = (int64_t(b) * p.heads_kv + h) * p.max_ctx;
      else if (p.layout == LA_KV_PACKED)
        u.row0 = int64_t(h) * cu[p.batch] + cu[b];
      else
        u.row0 = int64_t(b) * p.heads_kv + h;  // paged: rows come from the block table
      // request b's rows: (H_q, N_b) blocks, row (head j of the group, query i) = j N_b + i
      u.q_row = int32_t(cq[b] + int64_t(h) * rows + r0);
      u.rows = std::min(p.tile_rows, rows - r0);
      u.r0 = r0;
      u.nq = nq;
      u.iter_begin = int32_t(it);
      it += (int64_t(u.len) + tile_n - 1) / tile_n;   // C_n = ceil(n_b / T_n)   (Alg2§5)
      u.iter_end = int32_t(it);
      u.last_cta = u.host_cta = -1;
      units.push_back(u);
    }
  };
  if (p.layout != LA_KV_PACKED) {
    for (int b = 0; b < p.batch; ++b)           // batch -> heads -> context
      for (int h = 0; h < p.heads_kv; ++h) add(b, h);
  } else {
    for (int h = 0; h < p.heads_kv; ++h)        // heads -> total context
      for (int b = 0; b < p.batch; ++b) add(b, h);
  }
  total_iters = it;
}

void streamk_ranges(int64_t total_iters, int grid, std::vector<int32_t>& cta_begin) {
  // Reading C8: the first r = I mod G CTAs take ceil(I/G), the others floor(I/G).
  const int64_t q = total_iters / grid, r = total_iters % grid;
  cta_begin.resize(size_t(grid) + 1);
  for (int g = 0; g <= grid; ++g) cta_begin[g] = int32_t(g * q + std::min<int64_t>(g, r));
}

void weighted_ranges(int64_t total_iters, const std::vector<int32_t>& w, std::vector<int32_t>& cta_begin) {
  // SM-rate-weighted Eq. 2: one LeanTile per CTA plus a share of the other
  // R = I - G proportional to its weight, boundary g = min(g, I) + floor(R * W_{<g} / W) --
  // no empty range inside a unit (its host would wait for a partial nobody writes).  Integers
  // only (R < 2^31, W <= G * 2^20), so the oracle reproduces it exactly.
  const int64_t G = int64_t(w.size());
  int64_t W = 0;
  for (int32_t x : w) W += x;
  const int64_t R = std::max<int64_t>(total_iters - G, 0);
  cta_begin.resize(size_t(G) + 1);
  int64_t acc = 0;
  for (int64_t g = 0; g <= G; ++g) {
    cta_begin[size_t(g)] = int32_t(std::min(g, total_iters) + R * acc / W);
    if (g < G) acc += w[size_t(g)];
  }
}

void sequential_ranges(const std::vector<DevUnit>& units, std::vector<int32_t>& cta_begin) {
  cta_begin.resize(units.size() + 1);
  for (size_t u = 0; u < units.size(); ++u) cta_begin[u] = units[u].iter_begin;
  cta_begin[units.size()] = units.empty() ? 0 : units.back().iter_end;
}

void balanced_ranges(int64_t total_iters, int grid, int head_permille, int min_chunk, int max_chunks,
                     std::vector<int32_t>& cta_begin, std::vector<int32_t>& claim) {
  // B200-first extension: Alg. 2's equal ranges balance LeanTile COUNTS, but
  // per-SM streaming speed varies (measured 49-53 GB/s under equal work), so equal counts do
  // not finish together.  Every Eq. 2 range keeps its first ~head_permille / 1000 as a HEAD;
  // its last part is cut into k chunks of s LeanTiles that the persistent CTAs claim after
  // all heads, round by round over the ranges -- fast SMs take more chunks, and every unit's
  // last pieces are small.  Mirrors oracle.balanced_ranges bit for bit.
  cta_begin.assign(1, 0);
  std::vector<int32_t> heads;
  std::vector<std::vector<int32_t>> tails;
  const int64_t q = total_iters / grid, r = total_iters % grid;
  int32_t v = 0;
  for (int g = 0; g < grid; ++g) {
    const int64_t b = g * q + std::min<int64_t>(g, r), e = b + q + (g < r ? 1 : 0), L = e - b;
    if (L == 0) continue;
    const int64_t t0 = L * (1000 - head_permille) / 1000;
    const int64_t s = std::max<int64_t>(min_chunk, (t0 + max_chunks - 1) / max_chunks);
    const int64_t k = std::min(t0 / s, (L - 1) / s);  // the head keeps >= 1 LeanTile
    heads.push_back(v++);
    cta_begin.push_back(int32_t(e - k * s));
    std::vector<int32_t> chunks;
    for (int64_t j = 1; j <= k; ++j) {
      chunks.push_back(v++);
      cta_begin.push_back(int32_t(e - (k - j) * s));
    }
    tails.push_back(std::move(chunks));
  }
  claim = heads;
  size_t kmax = 0;
  for (const auto& t : tails) kmax = std::max(kmax, t.size());
  for (size_t j = 0; j < kmax; ++j)
    for (const auto& t : tails)
      if (j < t.size()) claim.push_back(t[j]);
}

void fixed_split_ranges(const std::vector<DevUnit>& units, int split, std::vector<int32_t>& cta_begin) {
  cta_begin.assign(1, 0);
  for (const DevUnit& u : units) {
    const int32_t cn = u.iter_end - u.iter_begin;
    const int32_t s = std::max(1, std::min<int32_t>(split, cn));
    const int32_t q = cn / s, r = cn % s;
    int32_t pos = u.iter_begin;
    for (int32_t j = 0; j < s; ++j) {
      pos += q + (j < r ? 1 : 0);
      cta_begin.push_back(pos);
    }
  }
}

int fa2_num_splits(int64_t units, int64_t max_cn, int sms) {
  if (units >= int64_t(0.8 * sms)) return 1;
  const int64_t max_s = std::min<int64_t>({128, int64_t(sms), max_cn});
  double best = 0.0;
  std::vector<double> eff(size_t(max_s) + 1, 0.0);
  for (int64_t s = 1; s <= max_s; ++s) {
    const double waves = double(units * s) / sms;
    eff[s] = waves / std::ceil(waves);
    best = std::max(best, eff[s]);
  }
  for (int64_t s = 1; s <= max_s; ++s)
    if (eff[s] >= 0.85 * best) return int(s);
  return 1;
}

static int owner_of(const std::vector<int32_t>& cta_begin, int64_t it) {
  // The CTA g with cta_begin[g] <= it < cta_begin[g+1]; empty CTAs (G > I) are skipped
  // because upper_bound lands past every CTA whose range starts at the same index.
  auto pos = std::upper_bound(cta_begin.begin(), cta_begin.end(), int32_t(it));
  return int(pos - cta_begin.begin()) - 1;
}

void finish_schedule(Schedule& s) {
  s.grid = int(s.cta_begin.size()) - 1;
  const int G = s.grid;
  for (DevUnit& u : s.units) {
    u.host_cta = owner_of(s.cta_begin, u.iter_begin);     // host block (Alg2§17)
    u.last_cta = owner_of(s.cta_begin, u.iter_end - 1);   // reading C9 of Alg2§26
  }
  s.cta_first_unit.assign(G, 0);
  size_t unit = 0;
  int64_t segs = 0, partials = 0;
  for (int g = 0; g < G; ++g) {
    const int64_t b = s.cta_begin[g], e = s.cta_begin[g + 1];
    while (unit < s.units.size() && s.units[unit].iter_end <= b) ++unit;
    s.cta_first_unit[g] = int32_t(std::min(unit, s.units.empty() ? 0 : s.units.size() - 1));
    size_t u = unit;
    for (int64_t it = b; it < e;) {                        // Alg2§10, §41 (reading C10)
      while (s.units[u].iter_end <= it) ++u;
      ++segs;
      if (it != s.units[u].iter_begin) ++partials;         // non-host segment (Alg2§19)
      it = s.units[u].iter_end;
    }
  }
  s.num_segments = segs;
  s.num_partials = partials;
}

void export_segments(const Schedule& s, std::vector<int32_t>& rows) {
  rows.clear();
  rows.reserve(size_t(s.num_segments) * 7);
  for (int g = 0; g < s.grid; ++g) {
    const int64_t cta_start = s.cta_begin[g], cta_end = s.cta_begin[g + 1];   // Alg2§9
    size_t u = size_t(s.cta_first_unit[g]);
    for (int64_t it = cta_start; it < cta_end;) {
      while (s.units[u].iter_end <= it) ++u;                                   // tile_idx §11
      const DevUnit& d = s.units[u];
      const int64_t tile_iter = d.iter_begin, tile_iter_end = d.iter_end;      // §12-13
      rows.push_back(g);
      rows.push_back(int32_t(u));
      rows.push_back(int32_t(it - tile_iter));                                 // local_iter §14
      rows.push_back(int32_t(std::min(tile_iter_end, cta_end) - tile_iter));   // §15
      rows.push_back(it == tile_iter ? 1 : 0);                                 // host §17
      rows.push_back(cta_end >= tile_iter_end ? 1 : 0);                        // finishing §18
      rows.push_back(d.last_cta);                                              // §26 (C9)
      it = tile_iter_end;                                                      // §41
    }
  }
}

}  // namespace la
