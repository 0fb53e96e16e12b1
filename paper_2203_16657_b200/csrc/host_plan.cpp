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
