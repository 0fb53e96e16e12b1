// Host-side planning helpers (native, O(nnz)) exported through the C ABI.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/commdyn_cuda.h"

// Reorder every row's intra run so that the 16-byte shared-memory gathers one
// 8-lane row group issues together (lane t reads entries 8t..8t+7 of each
// 64-entry block; instruction k touches entry 8t+k of every lane, i.e. one
// quarter-warp phase per (block, k)) hit distinct bank groups (column mod 8).
// Entries are counting-sorted by bank group and dealt round-robin over the
// row's phases, so equal bank groups land in different phases.  The sum a row
// produces is unchanged up to floating-point reassociation; the order is a
// deterministic function of the row.
extern "C" CDK_API int cdk_host_bank_order(uint16_t *cols, const int64_t *ptr, int64_t n_rows,
                                           int32_t pad_value, int32_t pad_bank) {
  if (!cols || !ptr || n_rows < 0) return CDK_INPUT;
  std::vector<uint16_t> vals, out;
  std::vector<int> cap, fill;
  for (int64_t r = 0; r < n_rows; ++r) {
    const int64_t a = ptr[r], b = ptr[r + 1];
    const int64_t L = b - a;
    if (L <= 8) continue;  // a single lane-chunk: one entry per phase already
    if (L % 8) return CDK_INPUT;
    vals.assign(cols + a, cols + b);
    // counting sort by bank group (pads carry the zero slot's bank)
    int cnt[9] = {0};
    for (uint16_t v : vals) cnt[(v == pad_value ? pad_bank : (v & 7)) + 1]++;
    for (int i = 0; i < 8; ++i) cnt[i + 1] += cnt[i];
    out.resize(L);
    for (uint16_t v : vals) out[cnt[v == pad_value ? pad_bank : (v & 7)]++] = v;
    // phases: block m (64 entries), instruction k -> lanes t < T_m
    const int64_t nblk = (L + 63) / 64;
    const int64_t P = 8 * nblk;
    cap.assign(P, 0);
    fill.assign(P, 0);
    for (int64_t m = 0; m < nblk; ++m) {
      const int64_t Lm = std::min<int64_t>(64, L - 64 * m);
      for (int k = 0; k < 8; ++k) cap[8 * m + k] = (int)(Lm / 8);
    }
    int64_t j = 0;
    for (int64_t s = 0; s < L; ++s) {
      while (fill[j] == cap[j]) j = (j + 1) % P;
      const int64_t m = j / 8, k = j % 8, t = fill[j]++;
      cols[a + 64 * m + 8 * t + k] = out[s];
      j = (j + 1) % P;
    }
  }
  return CDK_OK;
}

// Triangles {i < j < k} of an undirected graph given as a symmetric CSR with
// sorted global columns (no self loops).  Writes up to `cap` triangles as
// int32 triples to out (may be NULL) and returns the total count (or -1 on
// bad input).  O(sum over edges of min degree) via sorted-list intersection.
extern "C" CDK_API int64_t cdk_host_triangles(const int64_t *ptr, const int32_t *cols,
                                              int64_t n, int32_t *out, int64_t cap) {
  if (!ptr || (!cols && ptr[n] > 0) || n < 0) return -1;
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t *ni = cols + ptr[i], *ni_end = cols + ptr[i + 1];
    const int32_t *jt = std::upper_bound(ni, ni_end, (int32_t)i);
    for (; jt < ni_end; ++jt) {
      const int32_t j = *jt;
      // common neighbours k > j of i and j
      const int32_t *a = std::upper_bound(jt + 1 - 1, ni_end, j);
      const int32_t *b = std::upper_bound(cols + ptr[j], cols + ptr[j + 1], j);
      const int32_t *b_end = cols + ptr[j + 1];
      while (a < ni_end && b < b_end) {
        if (*a < *b) {
          ++a;
        } else if (*b < *a) {
          ++b;
        } else {
          if (out && count < cap) {
            out[3 * count] = (int32_t)i;
            out[3 * count + 1] = j;
            out[3 * count + 2] = *a;
          }
          ++count;
          ++a;
          ++b;
        }
      }
    }
  }
  return count;
}

// Lane-per-row sliced ("ELL") intra layout of the ELL stage kernel.  A warp
// owns one rblock (<= 32 rows, lane = row) and walks its rows in lockstep,
// one 16-byte chunk (8 uint16 columns) per lane per step group; every
// LDS.128 the warp issues is one entry per lane, served per quarter-warp
// (8 lanes = 8 rows, a "bundle").  The entries of each bundle are scheduled
// so that the 8 lanes of every step hit 8 distinct bank groups (column mod
// 8): the bundle's (row x bank-group) count matrix, padded to a Delta-regular
// bipartite multigraph (Delta = max(longest row, fullest bank group)), is
// split into Delta perfect matchings (Birkhoff / Koenig), each used for as
// many steps as its smallest cell allows.  Padding slots of staged rblocks
// point at the zero slot of their assigned bank group (zero_slot + g), so a
// padded step costs no extra wavefront; unstaged rblocks (global gathers)
// pad with CDK_INTRA_PAD (skipped).  Chunks per rblock = ceil(max Delta / 8).
//   ell_off[b]: start of rblock b in uint4 units; chunk c of lane l is
//   ell[(ell_off[b] + 32 c + l) * 8 .. +8).  ell == NULL: sizes only.
// Columns are taken from each row's run ptr[r]..ptr[r+1] (pads skipped) in
// ascending order; bank groups are (column + bank_shift[b]) mod 8, i.e. of
// the global node index when bank_shift is the column base mod 8, so the
// schedule is a deterministic function of the rows' global columns (the
// same before and after rebasing, and on every shard).
namespace {
struct BundleSched {
  int cnt[8][8];
  int m[8][8];
  int match_row[8], match_col[8];
  bool seen[8];
  bool augment(int r) {
    for (int g = 0; g < 8; ++g) {
      if (m[r][g] <= 0 || seen[g]) continue;
      seen[g] = true;
      if (match_col[g] < 0 || augment(match_col[g])) {
        match_col[g] = r;
        match_row[r] = g;
        return true;
      }
    }
    return false;
  }
  bool perfect() {
    for (int i = 0; i < 8; ++i) match_row[i] = match_col[i] = -1;
    for (int r = 0; r < 8; ++r) {
      for (int g = 0; g < 8; ++g) seen[g] = false;
      if (!augment(r)) return false;
    }
    return true;
  }
};
}  // namespace

extern "C" CDK_API int cdk_host_ell_intra(const int64_t *rblk_row0, int32_t n_rblk,
                                          const int64_t *ptr, const uint16_t *cols,
                                          const uint8_t *staged, const uint8_t *bank_shift,
                                          int32_t zero_slot, int64_t *ell_off, uint16_t *ell) {
  if (!rblk_row0 || !ptr || !staged || !ell_off || n_rblk < 0 || (zero_slot & 7)) return CDK_INPUT;
  const uint16_t PAD = 0xFFFFu;
  std::vector<uint16_t> lists[8][8];
  std::vector<uint16_t> seq[32];
  BundleSched bs;
  if (!ell) ell_off[0] = 0;
  for (int32_t b = 0; b < n_rblk; ++b) {
    const int64_t r0 = rblk_row0[b], r1 = rblk_row0[b + 1];
    if (r1 - r0 > 32 || r1 < r0) return CDK_INPUT;
    const int sh = bank_shift ? bank_shift[b] : 0;  // bank group = (column + sh) mod 8
    int delta[4] = {0, 0, 0, 0};
    int dmax = 0;
    for (int q = 0; q < 4; ++q) {
      int L[8] = {0}, C[8] = {0};
      for (int l = 0; l < 8; ++l) {
        const int64_t r = r0 + 8 * q + l;
        if (r >= r1) continue;
        for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
          const uint16_t v = cols[e];
          if (v == PAD) continue;
          ++L[l];
          ++C[(v + sh) & 7];
        }
      }
      int d = 0;
      for (int i = 0; i < 8; ++i) d = std::max(d, std::max(L[i], C[i]));
      delta[q] = d;
      dmax = std::max(dmax, d);
    }
    const int64_t nch = (dmax + 7) / 8;
    if (!ell) {
      ell_off[b + 1] = ell_off[b] + 32 * nch;
      continue;
    }
    if (ell_off[b + 1] - ell_off[b] != 32 * nch) return CDK_INPUT;
    const int steps = (int)(8 * nch);
    const bool st = staged[b] != 0;
    for (int q = 0; q < 4; ++q) {
      int L[8] = {0}, C[8] = {0};
      for (int l = 0; l < 8; ++l)
        for (int g = 0; g < 8; ++g) lists[l][g].clear();
      for (int l = 0; l < 8; ++l) {
        const int64_t r = r0 + 8 * q + l;
        if (r >= r1) continue;
        for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
          const uint16_t v = cols[e];
          if (v == PAD) continue;
          lists[l][(v + sh) & 7].push_back(v);
          ++L[l];
          ++C[(v + sh) & 7];
        }
      }
      for (int l = 0; l < 8; ++l) {
        std::sort(lists[l][0].begin(), lists[l][0].end());
        for (int g = 1; g < 8; ++g) std::sort(lists[l][g].begin(), lists[l][g].end());
      }
      // Delta-regular completion: padding counts with row sums Delta - L and
      // column sums Delta - C (northwest-corner fill)
      const int d = delta[q];
      int dr[8], dc[8];
      for (int i = 0; i < 8; ++i) {
        dr[i] = d - L[i];
        dc[i] = d - C[i];
      }
      for (int l = 0; l < 8; ++l)
        for (int g = 0; g < 8; ++g) {
          bs.cnt[l][g] = (int)lists[l][g].size();
          const int x = std::min(dr[l], dc[g]);
          bs.m[l][g] = bs.cnt[l][g] + x;
          dr[l] -= x;
          dc[g] -= x;
        }
      size_t take[8][8] = {};
      for (int l = 0; l < 8; ++l) seq[8 * q + l].clear();
      int k = 0;
      while (k < d) {
        if (!bs.perfect()) return CDK_NUMERIC;  // internal: schedule invariant broken
        int t = d - k;
        for (int l = 0; l < 8; ++l) t = std::min(t, bs.m[l][bs.match_row[l]]);
        for (int l = 0; l < 8; ++l) {
          const int g = bs.match_row[l];
          bs.m[l][g] -= t;
          for (int s = 0; s < t; ++s) {
            if (take[l][g] < lists[l][g].size()) {
              seq[8 * q + l].push_back(lists[l][g][take[l][g]++]);
            } else {
              seq[8 * q + l].push_back(st ? (uint16_t)(zero_slot + g) : PAD);
            }
          }
        }
        k += t;
      }
      for (int l = 0; l < 8; ++l) {  // steps beyond Delta: distinct bank groups per step
        for (int s = d; s < steps; ++s)
          seq[8 * q + l].push_back(st ? (uint16_t)(zero_slot + ((l + s) & 7)) : PAD);
        for (int g = 0; g < 8; ++g)
          if (take[l][g] != lists[l][g].size()) return CDK_NUMERIC;  // internal: schedule invariant broken
      }
    }
    uint16_t *dst = ell + ell_off[b] * 8;
    for (int64_t c = 0; c < nch; ++c)
      for (int l = 0; l < 32; ++l)
        for (int p = 0; p < 8; ++p) dst[(c * 32 + l) * 8 + p] = seq[l][c * 8 + p];
  }
  return CDK_OK;
}
