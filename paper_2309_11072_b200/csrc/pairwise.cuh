// pairwise.cuh -- numpy's float64 pairwise summation, restated for the GPU.
//
// numpy reduces a contiguous float64 array as 0.0 + pairwise(a, n) with
// (numpy/_core/src/umath/loops_utils.h pairwise_sum_DOUBLE):
//   n < 8     : sequential from 0.0
//   n <= 128  : 8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//               then the sequential tail
//   otherwise : n2 = n/2 - (n/2 % 8); pairwise(a, n2) + pairwise(a+n2, n-n2)
// Call sites on the hot path: np.mean in tone_map (tonemap.py:101) and
// x.sum() in fit_region (estimator.py:159).  Verified against numpy in
// tests/test_oracle.py (oracle/hdll_oracle.c ho_pairwise_sum).
//
// GPU form: the recursion tree is cut at depth L (pairwise_level); each
// depth-L node is summed sequentially by one thread (its subtree is exactly
// numpy's), and the 2^L node sums are combined by a perfect binary tree,
// which is the same sequence of `left + right` additions numpy performs.
#pragma once

#include "encoder.cuh"

namespace hdll {

// (offset, size) of node `idx` at depth L of the pairwise tree over n elements.
__host__ __device__ __forceinline__ void pairwise_node(long long n, int L, long long idx, long long* off, long long* size) {
  long long o = 0, m = n;
  for (int l = L - 1; l >= 0; l--) {
    long long n2 = m / 2;
    n2 -= n2 % 8;
    if ((idx >> l) & 1) {
      o += n2;
      m -= n2;
    } else {
      m = n2;
    }
  }
  *off = o;
  *size = m;
}

template <class Acc>
__device__ double pairwise_seq(const Acc& a, long long off, long long n) {
  if (n < 8) {
    double res = 0.;
    for (long long i = 0; i < n; i++) res += a(off + i);
    return res;
  } else if (n <= 128) {
    double r0 = a(off + 0), r1 = a(off + 1), r2 = a(off + 2), r3 = a(off + 3);
    double r4 = a(off + 4), r5 = a(off + 5), r6 = a(off + 6), r7 = a(off + 7);
    long long i;
    long long lim = n - (n % 8);
    for (i = 8; i < lim; i += 8) {
      r0 += a(off + i + 0);
      r1 += a(off + i + 1);
      r2 += a(off + i + 2);
      r3 += a(off + i + 3);
      r4 += a(off + i + 4);
      r5 += a(off + i + 5);
      r6 += a(off + i + 6);
      r7 += a(off + i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; i++) res += a(off + i);
    return res;
  } else {
    long long n2 = n / 2;
    n2 -= n2 % 8;
    double left = pairwise_seq(a, off, n2);
    return left + pairwise_seq(a, off + n2, n - n2);
  }
}

// One warp sums one pairwise subtree [off, off + n) exactly as pairwise_seq:
// the leaves (n <= 128) are found by the same recursion and summed four at a
// time by groups of 8 lanes -- lane j of a group is numpy's accumulator r[j],
// so every addition happens in numpy's order -- then lane 0 combines the leaf
// sums along the recursion tree.  Result in every lane.
//
// Every lane finds its own leaves by descending from the root with a table of
// leaf counts per subtree size; a leaf's path (bit q = went right at depth q)
// drives the combine, which keeps one pending left-sibling sum per depth in
// shared memory.
constexpr int kMaxLeaves = 160;  // n <= 8192

struct PwScratch {
  double leaf[kMaxLeaves];
  long long lo[kMaxLeaves];
  int ln[kMaxLeaves];         // size | depth << 16
  unsigned path[kMaxLeaves];  // bit q: went right at depth q
  double pending[32];
};

__device__ __forceinline__ long long pw_split(long long m) {
  const long long n2 = m / 2;
  return n2 - n2 % 8;
}

// Leaves of a subtree of m <= kPwTableN elements, by size (host-built table:
// pairwise_leaf_counts), so every lane can descend to its own leaf directly.
constexpr int kPwTableN = 8192;

__host__ __device__ inline void pairwise_leaf_counts(uint8_t* cnt /* kPwTableN + 1 */) {
  for (int m = 0; m <= kPwTableN; m++) {
    if (m <= 128) {
      cnt[m] = 1;
    } else {
      int n2 = m / 2;
      n2 -= n2 % 8;
      cnt[m] = (uint8_t)(cnt[n2] + cnt[m - n2]);
    }
  }
}

// one copy per translation unit that sums pairwise trees (fit.cu, tonemap.cu)
static __constant__ uint8_t c_pw_leaves[kPwTableN + 1];

static inline void upload_pw_table() {
  static uint8_t cnt[kPwTableN + 1];
  pairwise_leaf_counts(cnt);
  cudaMemcpyToSymbol(c_pw_leaves, cnt, sizeof(cnt));
}

// kTailLanes: a leaf's sequential tail is loaded by the lanes of its group
// together (cheap accessors: k_seg_nodes); otherwise lane 0 of the group
// reads it element by element (the tone map's accessor computes a log per read)
template <class Acc, bool kTailLanes = true>
__device__ double warp_pairwise(const Acc& a, long long off, long long n, PwScratch& sc) {
  const uint8_t* leaves_of = c_pw_leaves;
  const int lane = threadIdx.x & 31, grp = lane >> 3, j = lane & 7;
  const int nleaf = leaves_of[n];
  // every lane descends to its leaves: (offset, size), and the path / depth the combine needs
  for (int i = lane; i < nleaf; i += 32) {
    long long lo = off, m = n;
    int idx = i, depth = 0;
    unsigned path = 0;
    while (m > 128) {
      const long long n2 = pw_split(m);
      const int cl = leaves_of[n2];
      if (idx < cl) {
        m = n2;
      } else {
        idx -= cl;
        lo += n2;
        m -= n2;
        path |= 1u << depth;
      }
      depth++;
    }
    sc.lo[i] = lo;
    sc.ln[i] = (int)m | (depth << 16);
    sc.path[i] = path;
  }
  __syncwarp();
  for (int base = 0; base < nleaf; base += 4) {
    const int li = base + grp;
    const bool mine = li < nleaf;
    const long long lo = mine ? sc.lo[li] : 0, ln = mine ? (sc.ln[li] & 0xFFFF) : 0;
    const long long lim = ln - (ln % 8);
    double r = 0.0;
    // the sequential part (the tail past the last multiple of 8, or a whole
    // leaf under 8 samples): one element per lane of the group, loaded with
    // the rest instead of one dependent load per addition
    const long long tb = ln < 8 ? 0 : lim, tcnt = ln - tb;  // 0..7 elements
    double tv = 0.0;
    if (kTailLanes && mine && j < tcnt) tv = a(lo + tb + j);
    if (mine && ln >= 8) {
      // a leaf holds <= 128 samples: issue all 16 loads of the lane before the adds
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; q++) v[q] = (8 * q < lim) ? a(lo + 8 * q + j) : 0.0;
      r = v[0];
#pragma unroll
      for (int q = 1; q < 16; q++)
        if (8 * q < lim) r += v[q];
    }
    const double p2 = r + __shfl_down_sync(0xffffffffu, r, 1);    // r0+r1, r2+r3, ...
    const double q4 = p2 + __shfl_down_sync(0xffffffffu, p2, 2);  // (r0+r1)+(r2+r3), ...
    const double s8 = q4 + __shfl_down_sync(0xffffffffu, q4, 4);  // ((..)+(..))+((..)+(..))
    double res = ln < 8 ? 0.0 : s8;
    if constexpr (kTailLanes) {
#pragma unroll
      for (int t = 0; t < 7; t++) {  // numpy's sequential tail, in order
        const double x = __shfl_sync(0xffffffffu, tv, (lane & ~7) + t);
        if (t < tcnt) res += x;
      }
    } else if (mine && j == 0) {
      for (long long i = tb; i < ln; i++) res += a(lo + i);
    }
    if (mine && j == 0) sc.leaf[li] = res;
  }
  __syncwarp();
  double out = 0.0;
  if (lane == 0)
    for (int i = 0; i < nleaf; i++) {  // post-order combine: a right child completes its parent
      double v = sc.leaf[i];
      const unsigned path = sc.path[i];
      int dd = sc.ln[i] >> 16;
      while (dd > 0 && ((path >> (dd - 1)) & 1u)) {
        v = sc.pending[dd - 1] + v;
        dd--;
      }
      if (dd == 0) out = v;
      else sc.pending[dd - 1] = v;
    }
  __syncwarp();
  return __shfl_sync(0xffffffffu, out, 0);
}

// Perfect-binary-tree sum of vals[0 .. 2^L) by one CTA (blockDim.x = 256).
// Returns the result in thread 0.
__device__ __forceinline__ double tree_reduce_block(const double* vals, int L, double* smem /*256*/) {
  long long m = 1LL << L;
  int t = threadIdx.x;
  int nt = blockDim.x;  // power of two
  double v = 0.0;
  if (m >= nt) {
    // each thread reduces a perfect subtree of m/nt consecutive leaves with a
    // binary-counter stack (equal-height partials combine left + right)
    long long chunk = m / nt;
    double stk[40];
    int hgt[40];
    int sp = 0;
    for (long long i = 0; i < chunk; i++) {
      double x = vals[(long long)t * chunk + i];
      int hh = 0;
      while (sp > 0 && hgt[sp - 1] == hh) {
        x = stk[sp - 1] + x;
        sp--;
        hh++;
      }
      stk[sp] = x;
      hgt[sp] = hh;
      sp++;
    }
    v = stk[0];
    smem[t] = v;
    __syncthreads();
    for (int s = 1; s < nt; s <<= 1) {
      if ((t % (2 * s)) == 0) smem[t] = smem[t] + smem[t + s];
      __syncthreads();
    }
  } else {
    if (t < m) smem[t] = vals[t];
    __syncthreads();
    for (long long s = 1; s < m; s <<= 1) {
      if (t < m && (t % (2 * s)) == 0) smem[t] = smem[t] + smem[t + s];
      __syncthreads();
    }
  }
  return smem[0];
}

}  // namespace hdll
