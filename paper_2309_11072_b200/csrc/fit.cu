// fit.cu -- SLRME per-(channel, exponent) regression (estimator.py:145-214).
//
// For every channel c and exponent e present (ascending), the reference fits
// x = S*[E == e], y = M[E == e] in raster order with
//   sx = x.sum()        numpy pairwise sum              (estimator.py:159)
//   sy = y.sum()        exact (integer-valued)          (:160)
//   sxx = np.dot(x, x), sxy = np.dot(x, y)   OpenBLAS ddot (:161-162)
//   den = n*sxx - sx*sx; a = (n*sxy - sx*sy)/den; b = (sy - a*sx)/n, with the
//   degenerate fallback (0, sy/n)           (:163-169), then float32 RNE (:205-214).
// With sigma > 0 S* is real-valued and the float sums are order dependent, so
// the GPU follows the reference's order exactly:
//   1. stable counting sort of the (S*, M) samples by E (raster order inside a bin),
//      written contiguously so the sums below stream them;
//   2. pairwise tree for sx (pairwise.cuh) over each bin's sorted samples;
//   3. the OpenBLAS kernel's lane structure for sxx/sxy: 32 (SKYLAKEX) or 16
//      (HASWELL) sequential FMA chains, its fold order, its tail, and the
//      level-1 thread split (n > 10000) as a parameter (blas_threads);
//   4. the fit formula in fp64 and __double2float_rn.
// sy and the counts are exact integers (int64 atomics).
#include "encoder.cuh"
#include "pairwise.cuh"

namespace hdll {

constexpr int kSegs = 3 * 256;

// ---------------------------------------------------------------------------
// 1. stable counting sort by exponent
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sort_hist(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.fit_owner || d.hist_fused) return;
  const int tile = blockIdx.x;
  if (tile >= d.sort_tiles) return;
  __shared__ unsigned hist[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const long long p0 = (long long)tile * kSortTile;  // sample index; pixel fit_p0 + sample
  const uint32_t* px = reinterpret_cast<const uint32_t*>(d.rgbe) + d.fit_p0;
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  for (int k = threadIdx.x; k < kSortTile; k += blockDim.x) {
    const long long p = p0 + k;
    const bool valid = p < d.fit_m;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) continue;
    const unsigned e = px[p] >> 24;
    // warp-aggregated: one shared atomic per distinct exponent in the warp
    const unsigned peers = __match_any_sync(act, e);
    if ((peers & lt) == 0) atomicAdd(&hist[e], (unsigned)__popc(peers));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += blockDim.x) {
    d.tile_hist[(long long)e * d.sort_tiles + tile] = hist[e];
    if (hist[e]) atomicAdd(&d.bin_count[e], hist[e]);
  }
}

// bin starts + per-tile absolute offsets (in place over tile_hist, bin-major
// [256][sort_tiles]): one CTA per bin, threads scan contiguous runs of tiles
__global__ void __launch_bounds__(256) k_sort_scan(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.fit_owner || d.int_fit) return;
  const int e = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  __shared__ unsigned s_below, wsum[8];
  if (w == 0) {  // bin start: counts of the lower bins
    unsigned below = 0;
    for (int k = lane; k < e; k += 32) below += d.bin_count[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if (lane == 0) {
      s_below = below;
      d.bin_start[e] = below;
      if (e == 255) d.bin_start[256] = below + d.bin_count[255];
    }
  }
  // an empty bin's tile offsets are never read (k_sort_scatter places no sample in it)
  if (d.bin_count[e] == 0) return;
  const long long T = d.sort_tiles;
  unsigned* row = d.tile_hist + (long long)e * T;
  const long long per = (T + 255) / 256;
  const long long t0 = min(T, t * per), t1 = min(T, t0 + per);
  unsigned run = 0;
#pragma unroll 4
  for (long long k = t0; k < t1; k++) run += row[k];
  unsigned wt;
  unsigned off = warp_excl_sum(run, &wt);
  if (lane == 0) wsum[w] = wt;
  __syncthreads();
  for (int k = 0; k < w; k++) off += wsum[k];
  off += s_below;
  for (long long k = t0; k < t1; k++) {
    const unsigned c = row[k];
    row[k] = off;
    off += c;
  }
}

// Stable placement: within a tile the samples are first ranked and staged in
// shared memory in bin order, then written out so that consecutive threads
// store consecutive positions of a bin (coalesced).
struct ScatterSmem {
  double xw[3][kSortTile];  // the tile's S* window (full, aligned tiles: one bulk copy per channel)
  uint64_t bar;
  unsigned wcnt[8][256];
  unsigned loc_off[257];
  unsigned g_off[256];
  uint16_t src[kSortTile];  // slot -> sample of the tile
  uint8_t ys[3][kSortTile];
  uint8_t es[kSortTile];
};

__global__ void __launch_bounds__(256) k_sort_scatter(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.fit_owner || d.int_fit) return;
  const int tile = blockIdx.x;
  if (tile >= d.sort_tiles) return;
  extern __shared__ __align__(16) uint8_t sm_raw[];
  ScatterSmem& sm = *reinterpret_cast<ScatterSmem*>(sm_raw);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t0 = (long long)tile * kSortTile;
  const int tn = (int)min((long long)kSortTile, d.fit_m - t0);
  const long long pb = d.fit_p0;  // desc pixel of sample 0
  const uint32_t* px = reinterpret_cast<const uint32_t*>(d.rgbe) + pb;
  const long long m = d.fit_m;
  const bool real = d.sigma_milli != 0;
  if (d.global_regression) {  // whole planes in raster order: identity placement
    for (int k = threadIdx.x; k < tn; k += blockDim.x) {
      const long long p = t0 + k;
      const uint32_t q = px[p];
#pragma unroll
      for (int c = 0; c < 3; c++) {
        d.xs[(long long)c * m + p] =
            real ? d.sstar[(long long)c * d.n + pb + p] : (double)d.s_planes[(long long)c * d.n + pb + p];
        d.ys[(long long)c * m + p] = (uint8_t)((q >> (8 * c)) & 0xFF);
      }
    }
    return;
  }
  // A full tile's S* window (3 x 8 KB) comes in by bulk copies issued first,
  // so the DRAM stream overlaps the ranking below and the placement gathers
  // read shared memory instead of scattered global words.
  const double* xg[3];
#pragma unroll
  for (int c = 0; c < 3; c++) xg[c] = d.sstar + (long long)c * d.n + pb + t0;
  const bool bulk = tn == kSortTile && real &&
                    ((reinterpret_cast<uintptr_t>(xg[0]) | reinterpret_cast<uintptr_t>(xg[1]) |
                      reinterpret_cast<uintptr_t>(xg[2])) & 15) == 0;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&sm.bar, 3 * kSortTile * sizeof(double));
#pragma unroll
    for (int c = 0; c < 3; c++) bulk_g2s(&sm.xw[c][0], xg[c], kSortTile * sizeof(double), &sm.bar);
  }
  constexpr int kPerWarp = kSortTile / 8;
  constexpr int kSteps = kPerWarp / 32;
  const int wb = w * kPerWarp;
  const unsigned lt = (1u << lane) - 1u;
  // the warp's RGBE words, all loads in flight before the counters are cleared
  // (each used to be a dependent DRAM round trip per step); kept for the
  // placement pass, with the exponent groups
  uint32_t qv[kSteps];
  unsigned pv[kSteps];
#pragma unroll
  for (int step = 0; step < kSteps; step++) {
    const int k = wb + step * 32 + lane;
    qv[step] = k < tn ? __ldg(px + t0 + k) : 0u;
  }
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sm.wcnt[0][0])[i] = 0;
  __syncthreads();
#pragma unroll
  for (int step = 0; step < kSteps; step++) {
    const int k = wb + step * 32 + lane;
    const bool valid = k < tn;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    pv[step] = 0;
    if (valid) {
      const unsigned e = qv[step] >> 24;
      const unsigned peers = __match_any_sync(act, e);
      pv[step] = peers;
      if ((peers & lt) == 0) sm.wcnt[w][e] += __popc(peers);
    }
  }
  __syncthreads();
  {  // bin offsets inside the tile, per-warp bases, absolute bin offsets of the tile
    const int e = threadIdx.x;
    unsigned tot = 0;
    for (int k = 0; k < 8; k++) tot += sm.wcnt[k][e];
    unsigned wtot;
    unsigned ex = warp_excl_sum(tot, &wtot);
    __shared__ unsigned wsum[8];
    if (lane == 31) wsum[w] = ex + tot;
    __syncthreads();
    unsigned pre = 0;
    for (int k = 0; k < w; k++) pre += wsum[k];
    const unsigned off = pre + ex;
    sm.loc_off[e] = off;
    if (e == 255) sm.loc_off[256] = off + tot;
    sm.g_off[e] = tot ? d.tile_hist[(long long)e * d.sort_tiles + tile] : 0u;  // (bins of this tile only)
    unsigned run = off;
    for (int k = 0; k < 8; k++) {
      unsigned c = sm.wcnt[k][e];
      sm.wcnt[k][e] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int step = 0; step < kSteps; step++) {
    const int k = wb + step * 32 + lane;
    const bool valid = k < tn;
    unsigned e = 0, peers = 0;
    if (valid) {
      const uint32_t q = qv[step];
      e = q >> 24;
      peers = pv[step];
      const unsigned slot = sm.wcnt[w][e] + __popc(peers & lt);
#pragma unroll
      for (int c = 0; c < 3; c++) sm.ys[c][slot] = (uint8_t)((q >> (8 * c)) & 0xFF);
      sm.src[slot] = (uint16_t)k;
      sm.es[slot] = (uint8_t)e;
    }
    __syncwarp();
    if (valid && (peers & lt) == 0) sm.wcnt[w][e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (tn == kSortTile && real) {  // full tile: every gather in flight before the stores
    constexpr int kR = kSortTile / 256;
    double xv[kR][3];
    if (bulk) {
      mbar_wait(&sm.bar, 0);
#pragma unroll
      for (int r = 0; r < kR; r++) {
        const int q = sm.src[threadIdx.x + 256 * r];
#pragma unroll
        for (int c = 0; c < 3; c++) xv[r][c] = sm.xw[c][q];
      }
    } else {
#pragma unroll
      for (int r = 0; r < kR; r++) {
        const long long p = t0 + sm.src[threadIdx.x + 256 * r];
#pragma unroll
        for (int c = 0; c < 3; c++) xv[r][c] = d.sstar[(long long)c * d.n + pb + p];
      }
    }
#pragma unroll
    for (int r = 0; r < kR; r++) {
      const int q = threadIdx.x + 256 * r;
      const unsigned e = sm.es[q];
      const long long gpos = (long long)sm.g_off[e] + (q - sm.loc_off[e]);
#pragma unroll
      for (int c = 0; c < 3; c++) {
        d.xs[(long long)c * m + gpos] = xv[r][c];
        d.ys[(long long)c * m + gpos] = sm.ys[c][q];
      }
    }
    return;
  }
  for (int q = threadIdx.x; q < tn; q += blockDim.x) {
    const unsigned e = sm.es[q];
    const long long gpos = (long long)sm.g_off[e] + (q - sm.loc_off[e]);
    const long long p = t0 + sm.src[q];  // a gather inside the tile's window (L1)
#pragma unroll
    for (int c = 0; c < 3; c++) {
      d.xs[(long long)c * m + gpos] =
          real ? d.sstar[(long long)c * d.n + pb + p] : (double)d.s_planes[(long long)c * d.n + pb + p];
      d.ys[(long long)c * m + gpos] = sm.ys[c][q];
    }
  }
}

// ---------------------------------------------------------------------------
// 2. segments: (channel, bin) or (channel, whole plane) for global_regression
// ---------------------------------------------------------------------------
struct SegView {
  long long n, off;
  bool identity;
};

__device__ __forceinline__ SegView seg_view(const ImgDesc& d, int s) {
  int e = s & 255;
  SegView v;
  if (d.global_regression) {
    v.n = e == 0 ? d.fit_m : 0;
    v.off = 0;
    v.identity = true;
  } else {
    v.n = d.bin_count[e];
    v.off = d.bin_start[e];
    v.identity = false;
  }
  return v;
}

struct XAcc {  // x[i] = S*_c of the i-th sample of a segment (contiguous after the sort)
  const double* p;
  __device__ __forceinline__ double operator()(long long i) const { return p[i]; }
};

__device__ __forceinline__ XAcc x_acc(const ImgDesc& d, int c, const SegView& v) {
  return XAcc{d.xs + (long long)c * d.fit_m + v.off};
}

// one CTA of kSegs threads per image: each segment's tree depth, then an
// exclusive scan of the node counts (2^L per non-empty segment)
__global__ void __launch_bounds__(kSegs) k_seg_setup(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.x];
  if (!d.slrme || d.int_fit) return;
  const int s = threadIdx.x;
  const SegView v = seg_view(d, s);
  const int L = v.n > 0 ? pairwise_level(v.n) : 0;
  d.seg_level[s] = L;
  long long tot;
  const long long ex = warp_excl_sum(v.n > 0 ? (1LL << L) : 0LL, &tot);
  __shared__ long long wsum[kSegs / 32];
  const int w = s >> 5;
  if ((s & 31) == 0) wsum[w] = tot;
  __syncthreads();
  long long pre = 0;
  for (int k = 0; k < w; k++) pre += wsum[k];
  d.seg_node_off[s] = pre + ex;
  if (s == kSegs - 1) d.seg_node_off[kSegs] = pre + ex + (v.n > 0 ? (1LL << L) : 0LL);
}

// one warp per depth-L node of a segment's pairwise tree
// one warp per run of kNodesPerWarp consecutive depth-L nodes (of every
// segment in turn): the node -> segment lookup is one warp-parallel search
// per run, then a forward walk
constexpr int kNodesPerWarp = 8;

__global__ void __launch_bounds__(128) k_seg_nodes(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.int_fit) return;
  __shared__ PwScratch pw[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long g0 = ((long long)blockIdx.x * 4 + warp) * kNodesPerWarp;
  const long long gend = d.seg_node_off[kSegs];
  if (g0 >= gend) return;
  // s with off[s] <= g0 < off[s+1]: the last of 32 strided probes, then the
  // last of the 24 entries after it (kSegs = 32 x 24)
  constexpr int kStride = kSegs / 32;
  const unsigned b1 = __ballot_sync(0xffffffffu, d.seg_node_off[lane * kStride] <= g0);
  const int base = (31 - __clz(b1)) * kStride;
  const unsigned b2 = __ballot_sync(0xffffffffu, lane < kStride && d.seg_node_off[base + lane] <= g0);
  int s = base + 31 - __clz(b2);
  for (long long g = g0; g < min(g0 + kNodesPerWarp, gend); g++) {
    while (d.seg_node_off[s + 1] <= g) s++;  // (segments without nodes are passed over)
    SegView v = seg_view(d, s);
    long long off, sz;
    pairwise_node(v.n, d.seg_level[s], g - d.seg_node_off[s], &off, &sz);
    const double r = warp_pairwise(x_acc(d, s >> 8, v), off, sz, pw[warp]);
    if (lane == 0) d.seg_nodes[g] = r;
  }
}

// ---------------------------------------------------------------------------
// 3. OpenBLAS ddot models (oracle/hdll_oracle.c ddot_compute), one warp per
//    (segment, thread-chunk); both dots (x.x and x.y) in one sweep.
// ---------------------------------------------------------------------------
struct MAcc {  // y[i] = M_c of the i-th sample of a segment
  const uint8_t* p;
  __device__ __forceinline__ double operator()(long long i) const { return (double)p[i]; }
};

template <class XA, class YA>
__device__ void warp_ddot2(const XA& X, const YA& Y, long long start, long long len, int kernel, double* out_xx,
                           double* out_xy) {
  const int lane = threadIdx.x & 31;
  long long n1 = len & ~15LL;
  double dxx = 0.0, dxy = 0.0;
  if (kernel == 0) {  // SKYLAKEX
    long long n32 = n1 & ~31LL;
    double axx = 0.0, axy = 0.0;
    long long i = lane;
    // the lane's chain is sequential; keep kPF loads in flight ahead of it
    constexpr int kPF = 16;
    for (; i + 32LL * (kPF - 1) < n32; i += 32LL * kPF) {
      double xv[kPF], yv[kPF];
#pragma unroll
      for (int u = 0; u < kPF; u++) {
        xv[u] = X(start + i + 32LL * u);
        yv[u] = Y(start + i + 32LL * u);
      }
#pragma unroll
      for (int u = 0; u < kPF; u++) {
        axx = __fma_rn(xv[u], xv[u], axx);
        axy = __fma_rn(xv[u], yv[u], axy);
      }
    }
    for (; i < n32; i += 32) {
      double x = X(start + i), y = Y(start + i);
      axx = __fma_rn(x, x, axx);
      axy = __fma_rn(x, y, axy);
    }
    // fold 512 -> 256: lane 8k+l (l < 4) holds acc[8k+l] + acc[8k+l+4]
    double fxx = axx + __shfl_down_sync(0xffffffffu, axx, 4);
    double fxy = axy + __shfl_down_sync(0xffffffffu, axy, 4);
    // 256-bit loop over [n32, n1): four 4-lane accumulators, 16 elements per step
    if ((lane & 7) < 4) {
      int k = lane >> 3, l = lane & 7;
      for (long long i = n32; i < n1; i += 16) {
        double x = X(start + i + 4 * k + l), y = Y(start + i + 4 * k + l);
        fxx = __fma_rn(x, x, fxx);
        fxy = __fma_rn(x, y, fxy);
      }
    }
    // s[l] = ((a0[l] + a1[l]) + a2[l]) + a3[l]; dot = (s0 + s2) + (s1 + s3)
    double s_xx[4], s_xy[4];
#pragma unroll
    for (int l = 0; l < 4; l++) {
      double v0 = __shfl_sync(0xffffffffu, fxx, l), v1 = __shfl_sync(0xffffffffu, fxx, 8 + l);
      double v2 = __shfl_sync(0xffffffffu, fxx, 16 + l), v3 = __shfl_sync(0xffffffffu, fxx, 24 + l);
      s_xx[l] = ((v0 + v1) + v2) + v3;
      v0 = __shfl_sync(0xffffffffu, fxy, l);
      v1 = __shfl_sync(0xffffffffu, fxy, 8 + l);
      v2 = __shfl_sync(0xffffffffu, fxy, 16 + l);
      v3 = __shfl_sync(0xffffffffu, fxy, 24 + l);
      s_xy[l] = ((v0 + v1) + v2) + v3;
    }
    if (n1) {
      dxx = (s_xx[0] + s_xx[2]) + (s_xx[1] + s_xx[3]);
      dxy = (s_xy[0] + s_xy[2]) + (s_xy[1] + s_xy[3]);
    }
    if (lane == 0)  // tail: dot = fma(y, x, dot)
      for (long long i = n1; i < len; i++) {
        double x = X(start + i), y = Y(start + i);
        dxx = __fma_rn(x, x, dxx);
        dxy = __fma_rn(y, x, dxy);
      }
  } else {  // HASWELL: 16 lanes, lane 4k+l = acc[k][l]
    double axx = 0.0, axy = 0.0;
    if (lane < 16) {
      long long i = lane;
      constexpr int kPF = 16;
      for (; i + 16LL * (kPF - 1) < n1; i += 16LL * kPF) {
        double xv[kPF], yv[kPF];
#pragma unroll
        for (int u = 0; u < kPF; u++) {
          xv[u] = X(start + i + 16LL * u);
          yv[u] = Y(start + i + 16LL * u);
        }
#pragma unroll
        for (int u = 0; u < kPF; u++) {
          axx = __fma_rn(xv[u], xv[u], axx);
          axy = __fma_rn(xv[u], yv[u], axy);
        }
      }
      for (; i < n1; i += 16) {
        double x = X(start + i), y = Y(start + i);
        axx = __fma_rn(x, x, axx);
        axy = __fma_rn(x, y, axy);
      }
    }
    double a[16], b[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
      a[j] = __shfl_sync(0xffffffffu, axx, j);
      b[j] = __shfl_sync(0xffffffffu, axy, j);
    }
    if (n1) {
      double t0[4], t1[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        t0[k] = a[4 * k + 0] + a[4 * k + 2];
        t1[k] = a[4 * k + 1] + a[4 * k + 3];
      }
      double u0 = t0[0] + t0[1], u1 = t1[0] + t1[1], v0 = t0[2] + t0[3], v1 = t1[2] + t1[3];
      dxx = (u0 + v0) + (u1 + v1);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        t0[k] = b[4 * k + 0] + b[4 * k + 2];
        t1[k] = b[4 * k + 1] + b[4 * k + 3];
      }
      u0 = t0[0] + t0[1];
      u1 = t1[0] + t1[1];
      v0 = t0[2] + t0[3];
      v1 = t1[2] + t1[3];
      dxy = (u0 + v0) + (u1 + v1);
    }
    if (lane == 0)  // tail without fma
      for (long long i = n1; i < len; i++) {
        double x = X(start + i), y = Y(start + i);
        dxx = dxx + x * x;
        dxy = dxy + y * x;
      }
  }
  *out_xx = dxx;
  *out_xy = dxy;
}

// The ddot lanes are sequential FMA chains (the reference's order), so the
// samples are streamed through shared memory with bulk async copies
// (cp.async.bulk + mbarrier, kStages deep) and each lane's chain only waits on
// FMA latency.  Blocks hold kBlk samples; the bulk region is [0, nmain) with
// nmain = n32 (SKYLAKEX, 32 lanes) or n1 (HASWELL, 16 lanes).
// 2 stages of 1024 samples (18.5 KB, twelve warps per SM): measured against
// 4 x 2048 (74 KB, three warps per SM), 4 x 1024 and 4 x 512 on config 1 at
// the 1- and 16-thread parity models and on config 3 at 16 threads: with 16
// OpenBLAS threads most bins of a batch split into 16 short chunks, whose
// warps are latency-bound, so resident warps count more than depth
// (config 1 fit 4.85 -> 3.37 ms at 16 threads, 3.04 -> 2.95 at 1; config 3
// 0.88 -> 0.95 ms).
#ifndef HDLL_DOT_BLK  // experiment builds: samples per staged block / pipeline depth
#define HDLL_DOT_BLK 1024
#endif
#ifndef HDLL_DOT_STAGES
#define HDLL_DOT_STAGES 2
#endif
constexpr int kBlk = HDLL_DOT_BLK, kStages = HDLL_DOT_STAGES;
struct DotSmem {
  uint64_t bar[kStages];
  double x[kStages][kBlk + 2];
  uint8_t y[kStages][kBlk + 32];
};

// A launch over a batch (launch_fit_bins: >= 8 images) has one warp per
// segment, which streams all its OpenBLAS chunks in turn through one
// continuous pipeline; a launch over fewer images spreads every segment's
// chunks over the grid's z, one warp each.  Config 1 at 16 threads: fit 3.37
// ms with a warp per chunk, 2.98 with a warp per segment (the grid's 16x more,
// mostly empty CTAs alone cost 0.28 ms); config 3 needs the parallel chunks
// (fit 0.93 ms, against 1.35 with one warp per segment below 1 Mi samples).

// Position in OpenBLAS's level-1 split of a segment of n samples into T
// chunks (width = ceil(rem / (T - used)), oracle/hdll_oracle.c ddot_compute):
// chunk u's start and width, its bulk region [0, nmain) and staged blocks.
// A warp visits chunks j0, j0 + G, j0 + 2G, ...
struct ChunkCursor {
  long long n, start, rem, width, nmain, nblk;
  int T, G, u, kernel;
  __device__ __forceinline__ void geom() {
    width = (rem + (T - u) - 1) / (T - u);
    if (width > rem) width = rem;
    const long long n1 = width & ~15LL;
    nmain = kernel == 0 ? (n1 & ~31LL) : n1;
    nblk = (nmain + kBlk - 1) / kBlk;
  }
  __device__ __forceinline__ void step() {  // to chunk u + 1
    start += width;
    rem -= width;
    u++;
    if (u < T) geom();
  }
  __device__ __forceinline__ void init(long long nn, int TT, int j0, int GG, int kern) {
    n = nn, T = TT, G = GG, kernel = kern;
    start = 0, rem = n, u = 0;
    geom();
    for (int k = 0; k < j0 && u < T; k++) step();
  }
  __device__ __forceinline__ bool next() {  // to chunk u + G; false past the last
    for (int k = 0; k < G && u < T; k++) step();
    return u < T;
  }
};

// grid: (kSegs, nimg, max chunks); one warp per (segment, OpenBLAS thread-chunk)
__global__ void __launch_bounds__(32) k_seg_dot(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.int_fit) return;
  const int s = blockIdx.x;
  SegView v = seg_view(d, s);
  if (v.n == 0) return;
  extern __shared__ __align__(16) uint8_t dot_raw[];
  DotSmem& sm = *reinterpret_cast<DotSmem*>(dot_raw);
  const int lane = threadIdx.x & 31;
  const int c = s >> 8;
  const XAcc X = x_acc(d, c, v);
  const MAcc M{d.ys + (long long)c * d.fit_m + v.off};
  const int T = (v.n > 10000 && d.blas_threads > 1) ? min(d.blas_threads, kMaxBlasThreads) : 1;
  if (lane == 0)
    for (int k = 0; k < kStages; k++) mbar_init(&sm.bar[k], 1);
  fence_mbar_init();
  __syncwarp();
  unsigned phase_bits = 0;  // parity of every stage's barrier, flipped at each consumed block
  // The warp's chunks j0, j0 + G, ... stream through one continuous pipeline
  // (the producer runs ahead across chunk boundaries).
  const int G = (int)gridDim.z;
  if ((int)blockIdx.z >= G || (int)blockIdx.z >= T) return;  // no chunk for this warp
  const int kernel = d.blas_kernel;
  ChunkCursor pc, cc;  // producer (lane 0) and consumer positions
  pc.init(v.n, T, (int)blockIdx.z, G, kernel);
  cc = pc;
  long long pb = 0, fp = 0, fc = 0;  // producer's block in its chunk; flat blocks issued / consumed
  auto issue_next = [&]() {  // the next block in flat order into stage fp % kStages, if any
    while (pb >= pc.nblk) {
      if (!pc.next()) return;
      pb = 0;
    }
    const int st = (int)(fp % kStages);
    const long long e0 = pb * kBlk, len = min((long long)kBlk, pc.nmain - e0);
    const char* xa = reinterpret_cast<const char*>(X.p + pc.start + e0);
    const char* xa0 = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(xa) & ~uintptr_t(15));
    const unsigned xbytes = (unsigned)(((xa - xa0) + len * 8 + 15) & ~15LL);
    const char* ya = reinterpret_cast<const char*>(M.p + pc.start + e0);
    const char* ya0 = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(ya) & ~uintptr_t(15));
    const unsigned ybytes = (unsigned)(((ya - ya0) + len + 15) & ~15LL);
    fence_proxy_async_smem();
    mbar_expect_tx(&sm.bar[st], xbytes + ybytes);
    bulk_g2s(&sm.x[st][0], xa0, xbytes, &sm.bar[st]);
    bulk_g2s(&sm.y[st][0], ya0, ybytes, &sm.bar[st]);
    pb++;
    fp++;
  };
  if (lane == 0)
    for (int k = 0; k < kStages - 1; k++) issue_next();
  __syncwarp();
  const int nl = kernel == 0 ? 32 : 16;  // lanes of the main loop
  do {
    const int j = cc.u;
    const long long start = cc.start, width = cc.width, nmain = cc.nmain, nblk = cc.nblk;
    const long long n1 = width & ~15LL;
    double axx = 0.0, axy = 0.0;
    unsigned long long sy = 0;
    for (long long b = 0; b < nblk; b++) {
      if (lane == 0) issue_next();  // keeps kStages - 1 blocks in flight, across chunks
      const int st = (int)(fc % kStages);
      fc++;
      mbar_wait(&sm.bar[st], (phase_bits >> st) & 1u);
      phase_bits ^= 1u << st;
      const long long e0 = b * kBlk, len = min((long long)kBlk, nmain - e0);
      const int mx = (int)((reinterpret_cast<uintptr_t>(X.p + start + e0) & 15) >> 3);
      const int my = (int)(reinterpret_cast<uintptr_t>(M.p + start + e0) & 15);
      const double* xs = &sm.x[st][mx];
      const uint8_t* ys = &sm.y[st][my];
      if (lane < nl) {
        unsigned sy32 = 0;  // a block's byte sum fits 32 bits: one add per sample
#pragma unroll 8
        for (int k = lane; k < (int)len; k += nl) {
          const unsigned yb = ys[k];
          const double x = xs[k], y = (double)yb;
          axx = __fma_rn(x, x, axx);
          axy = __fma_rn(x, y, axy);
          sy32 += yb;
        }
        sy += sy32;
      }
      __syncwarp();
    }
    // fold and tails (oracle/hdll_oracle.c ddot_compute)
    double dxx = 0.0, dxy = 0.0;
    if (kernel == 0) {
      double fxx = axx + __shfl_down_sync(0xffffffffu, axx, 4);  // 512 -> 256 fold
      double fxy = axy + __shfl_down_sync(0xffffffffu, axy, 4);
      if ((lane & 7) < 4) {
        const int k = lane >> 3, l = lane & 7;
        for (long long i = nmain; i < n1; i += 16) {
          const double x = X(start + i + 4 * k + l), y = M(start + i + 4 * k + l);
          fxx = __fma_rn(x, x, fxx);
          fxy = __fma_rn(x, y, fxy);
        }
      }
      double sxx4[4], sxy4[4];
#pragma unroll
      for (int l = 0; l < 4; l++) {
        double v0 = __shfl_sync(0xffffffffu, fxx, l), v1 = __shfl_sync(0xffffffffu, fxx, 8 + l);
        double v2 = __shfl_sync(0xffffffffu, fxx, 16 + l), v3 = __shfl_sync(0xffffffffu, fxx, 24 + l);
        sxx4[l] = ((v0 + v1) + v2) + v3;
        v0 = __shfl_sync(0xffffffffu, fxy, l);
        v1 = __shfl_sync(0xffffffffu, fxy, 8 + l);
        v2 = __shfl_sync(0xffffffffu, fxy, 16 + l);
        v3 = __shfl_sync(0xffffffffu, fxy, 24 + l);
        sxy4[l] = ((v0 + v1) + v2) + v3;
      }
      if (n1) {
        dxx = (sxx4[0] + sxx4[2]) + (sxx4[1] + sxx4[3]);
        dxy = (sxy4[0] + sxy4[2]) + (sxy4[1] + sxy4[3]);
      }
      if (lane == 0)
        for (long long i = n1; i < width; i++) {
          const double x = X(start + i), y = M(start + i);
          dxx = __fma_rn(x, x, dxx);
          dxy = __fma_rn(y, x, dxy);
        }
    } else {
      double a[16], bb[16];
#pragma unroll
      for (int q = 0; q < 16; q++) {
        a[q] = __shfl_sync(0xffffffffu, axx, q);
        bb[q] = __shfl_sync(0xffffffffu, axy, q);
      }
      if (n1) {
        double t0[4], t1[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          t0[k] = a[4 * k + 0] + a[4 * k + 2];
          t1[k] = a[4 * k + 1] + a[4 * k + 3];
        }
        double u0 = t0[0] + t0[1], u1 = t1[0] + t1[1], v0 = t0[2] + t0[3], v1 = t1[2] + t1[3];
        dxx = (u0 + v0) + (u1 + v1);
#pragma unroll
        for (int k = 0; k < 4; k++) {
          t0[k] = bb[4 * k + 0] + bb[4 * k + 2];
          t1[k] = bb[4 * k + 1] + bb[4 * k + 3];
        }
        u0 = t0[0] + t0[1];
        u1 = t1[0] + t1[1];
        v0 = t0[2] + t0[3];
        v1 = t1[2] + t1[3];
        dxy = (u0 + v0) + (u1 + v1);
      }
      if (lane == 0)
        for (long long i = n1; i < width; i++) {
          const double x = X(start + i), y = M(start + i);
          dxx = dxx + x * x;
          dxy = dxy + y * x;
        }
    }
    // y.sum() is an exact integer sum (estimator.py:160): any order
    for (long long i = nmain + lane; i < width; i += 32) sy += M.p[start + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sy += __shfl_xor_sync(0xffffffffu, sy, o);
    if (lane == 0) {
      d.dot_part[((long long)s * kMaxBlasThreads + j) * 2 + 0] = dxx;
      d.dot_part[((long long)s * kMaxBlasThreads + j) * 2 + 1] = dxy;
      atomicAdd(reinterpret_cast<unsigned long long*>(&d.sum_y[s]), sy);
    }
  } while (cc.next());
}

// ---------------------------------------------------------------------------
// 4. coefficients (fit_region, estimator.py:145-169) -> float32 table
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_seg_reduce_coef(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.slrme || d.int_fit) return;
  const int s = blockIdx.x;
  SegView v = seg_view(d, s);
  if (v.n == 0) return;
  __shared__ double sm[256];
  double sx = tree_reduce_block(d.seg_nodes + d.seg_node_off[s], d.seg_level[s], sm);
  if (threadIdx.x != 0) return;
  sx = 0.0 + sx;
  const int c = s >> 8;
  const long long sy_i = d.sum_y[s];  // global_regression: the (c, 0) segment spans the whole plane
  const double sy = (double)sy_i;
  const int T = (v.n > 10000 && d.blas_threads > 1) ? min(d.blas_threads, kMaxBlasThreads) : 1;
  double sxx = 0.0, sxy = 0.0;
  for (int j = 0; j < T; j++) {  // OpenBLAS: dot = dot + partial_j
    sxx = sxx + d.dot_part[((long long)s * kMaxBlasThreads + j) * 2 + 0];
    sxy = sxy + d.dot_part[((long long)s * kMaxBlasThreads + j) * 2 + 1];
  }
  sxx = 0.0 + sxx;  // numpy DOUBLE_dot: sum = 0.0; sum += cblas_ddot(...)
  sxy = 0.0 + sxy;
  const double dn = (double)v.n;
  double a = 0.0, b = sy / dn;
  double den = dn * sxx - sx * sx;
  if (den > 0.0) {
    double aa = (dn * sxy - sx * sy) / den;
    double bb = (sy - aa * sx) / dn;
    if (isfinite(aa) && isfinite(bb)) {
      a = aa;
      b = bb;
    }
  }
  float a32 = __double2float_rn(a), b32 = __double2float_rn(b);
  if (d.global_regression) {
    for (int e = 0; e < 256; e++) {
      d.a32[c * 256 + e] = a32;
      d.b32[c * 256 + e] = b32;
    }
  } else {
    d.a32[s] = a32;
    d.b32[s] = b32;
  }
  if (!isfinite(a32) || !isfinite(b32)) atomicOr(d.status, kErrNonFinite);
}

// ---------------------------------------------------------------------------
// sigma = 0 (north_star item 3): S* = S is an integer
// plane, so every sum of fit_region (estimator.py:159-162) is an exact integer
// below 2^53 whatever the order -- numpy's pairwise x.sum() and OpenBLAS's ddot
// (FMA of integer products) included.  No sort.  Every CTA privatises
// per-(channel, exponent) bins of sum x, sum y, sum x^2, sum x*y in shared
// memory, 32-bit (12 KB, so eight CTAs fit an SM): the CTA flushes them every
// kIntChunk pixels, and 255^2 * kIntChunk < 2^32.  Every pixel adds to its
// bins with native 32-bit shared atomics (lanes of a warp sharing an exponent
// collide on an address a few ways; warp-aggregating with match + reduce over
// partial masks measured slower: config 1 fit 11.2 ms, c3 1.8 ms).  A flush adds
// the CTA's non-zero bins into the image's int64 table with global atomics.
// The coefficients then follow the reference's fp64 formula from the exact
// sums (k_fit_int_coef), bit-identical to the order-replicating path.
// ---------------------------------------------------------------------------
constexpr int kIntThreads = 256;
constexpr int kIntChunk = kIntThreads * 64;  // pixels per CTA between flushes
static_assert(255ull * 255ull * kIntChunk < (1ull << 32), "32-bit bins cannot overflow between flushes");

__device__ __forceinline__ void int_bins_add(unsigned* W, unsigned key, const unsigned (&x)[3], uint32_t q) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const unsigned y = (q >> (8 * c)) & 0xFFu;
    atomicAdd(&W[(c * 4 + 0) * 256 + key], x[c]);
    atomicAdd(&W[(c * 4 + 1) * 256 + key], y);
    atomicAdd(&W[(c * 4 + 2) * 256 + key], x[c] * x[c]);
    atomicAdd(&W[(c * 4 + 3) * 256 + key], x[c] * y);
  }
}

__global__ void __launch_bounds__(kIntThreads) k_fit_int(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.int_fit) return;
  __shared__ unsigned W[12 * 256];  // [channel * 4 + (sum x, sum y, sum x^2, sum x*y)][exponent]
  for (int i = threadIdx.x; i < 12 * 256; i += kIntThreads) W[i] = 0u;
  __syncthreads();
  const bool global = d.global_regression != 0;
  // the fit samples: desc pixels [fit_p0, fit_p0 + fit_m) (a row band's own rows)
  const long long n = d.fit_m, plane = d.n;
  const uint32_t* px = reinterpret_cast<const uint32_t*>(d.rgbe) + d.fit_p0;
  const uint8_t* S = d.s_planes + d.fit_p0;
  // four pixels per thread and step, as one 16-byte RGBE load and one 4-byte
  // load per S plane when the planes' quads are aligned
  const bool vec = ((d.fit_p0 | plane) & 3) == 0;
  unsigned long long* isum = reinterpret_cast<unsigned long long*>(d.isum);
  unsigned long long* sumy = reinterpret_cast<unsigned long long*>(d.sum_y);
  const long long nchunks = (n + kIntChunk - 1) / kIntChunk;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long p1 = min(n, (ch + 1) * kIntChunk);
    for (long long p = ch * kIntChunk + 4LL * threadIdx.x; p < p1; p += 4LL * kIntThreads) {
      if (vec && p + 4 <= p1) {
        const uint4 q4 = __ldg(reinterpret_cast<const uint4*>(px + p));
        uint32_t sw[3];
#pragma unroll
        for (int c = 0; c < 3; c++) sw[c] = __ldg(reinterpret_cast<const uint32_t*>(S + (long long)c * plane + p));
        const uint32_t qs[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const unsigned x[3] = {(sw[0] >> (8 * k)) & 0xFFu, (sw[1] >> (8 * k)) & 0xFFu, (sw[2] >> (8 * k)) & 0xFFu};
          int_bins_add(W, global ? 0u : (qs[k] >> 24), x, qs[k]);  // global_regression: one (c, 0) segment
        }
      } else {
        for (long long pp = p; pp < min(p + 4, p1); pp++) {
          const uint32_t q = __ldg(px + pp);
          const unsigned x[3] = {__ldg(S + pp), __ldg(S + plane + pp), __ldg(S + 2 * plane + pp)};
          int_bins_add(W, global ? 0u : (q >> 24), x, q);
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 12 * 256; i += kIntThreads) {  // flush the non-zero bins into the int64 table
      const unsigned v = W[i];
      if (!v) continue;
      W[i] = 0u;
      const int k = i >> 8, e = i & 255, c = k >> 2, j = k & 3;
      const int seg = c * 256 + e;
      if (j == 1) atomicAdd(sumy + seg, (unsigned long long)v);
      else atomicAdd(isum + 3 * seg + (j == 0 ? 0 : j - 1), (unsigned long long)v);
    }
    __syncthreads();
  }
}

// fit_region (estimator.py:145-169) from the exact sums, one thread per segment
__global__ void __launch_bounds__(256) k_fit_int_coef(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (!d.int_fit) return;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= kSegs) return;
  const int c = s >> 8, e = s & 255;
  long long nn = 0;
  if (!d.global_regression) {
    nn = d.bin_count[e];
  } else if (e == 0) {  // the whole plane: every bin's samples
    for (int k = 0; k < 256; k++) nn += d.bin_count[k];
  }
  if (nn == 0) return;
  const long long* g = d.isum + 3 * s;
  const double sx = (double)g[0], sxx = (double)g[1], sxy = (double)g[2];  // exact: < 2^53
  const double sy = (double)d.sum_y[s];
  const double dn = (double)nn;
  double a = 0.0, b = sy / dn;
  const double den = dn * sxx - sx * sx;
  if (den > 0.0) {
    const double aa = (dn * sxy - sx * sy) / den;
    const double bb = (sy - aa * sx) / dn;
    if (isfinite(aa) && isfinite(bb)) {
      a = aa;
      b = bb;
    }
  }
  const float a32 = __double2float_rn(a), b32 = __double2float_rn(b);
  if (d.global_regression) {
    for (int k = 0; k < 256; k++) {
      d.a32[c * 256 + k] = a32;
      d.b32[c * 256 + k] = b32;
    }
  } else {
    d.a32[s] = a32;
    d.b32[s] = b32;
  }
  if (!isfinite(a32) || !isfinite(b32)) atomicOr(d.status, kErrNonFinite);
}

void launch_fit_int_sums(const ImgDesc* d_descs, int nimg, long long max_n, cudaStream_t st) {
  // one CTA per chunk, about 8 CTAs (12 KB of bins each) per SM over the batch
  long long gx = (max_n + kIntChunk - 1) / kIntChunk;
  const long long cap = (148 * 8 + nimg - 1) / nimg;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  k_fit_int<<<dim3((unsigned)gx, nimg), kIntThreads, 0, st>>>(d_descs);
}

void launch_fit_int_coef(const ImgDesc* d_descs, int nimg, cudaStream_t st) {
  k_fit_int_coef<<<dim3(kSegs / 256, nimg), 256, 0, st>>>(d_descs);
}

void launch_fit_int(const ImgDesc* d_descs, int nimg, long long max_n, cudaStream_t st) {
  launch_fit_int_sums(d_descs, nimg, max_n, st);
  launch_fit_int_coef(d_descs, nimg, st);
}

void launch_fit_hist(const ImgDesc* d_descs, int nimg, int max_sort_tiles, cudaStream_t st) {
  k_sort_hist<<<dim3(max_sort_tiles, nimg), 256, 0, st>>>(d_descs);
}

void launch_fit_sort(const ImgDesc* d_descs, int nimg, int max_sort_tiles, cudaStream_t st, bool any_hist) {
  if (any_hist) k_sort_hist<<<dim3(max_sort_tiles, nimg), 256, 0, st>>>(d_descs);
  k_sort_scan<<<dim3(256, nimg), 256, 0, st>>>(d_descs);
  cudaFuncSetAttribute(k_sort_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ScatterSmem));
  k_sort_scatter<<<dim3(max_sort_tiles, nimg), 256, sizeof(ScatterSmem), st>>>(d_descs);
}

void launch_fit_bins(const ImgDesc* d_descs, int nimg, long long max_nodes, int max_chunks, cudaStream_t st) {
  k_seg_setup<<<nimg, kSegs, 0, st>>>(d_descs);
  k_seg_nodes<<<dim3((unsigned)((max_nodes + 4 * kNodesPerWarp - 1) / (4 * kNodesPerWarp)), nimg), 128, 0, st>>>(d_descs);
  cudaFuncSetAttribute(k_seg_dot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DotSmem));
  const int zd = nimg >= 8 ? 1 : max_chunks;  // batches: a warp per segment; else a warp per chunk
  k_seg_dot<<<dim3(kSegs, nimg, zd), 32, sizeof(DotSmem), st>>>(d_descs);
  k_seg_reduce_coef<<<dim3(kSegs, nimg), 256, 0, st>>>(d_descs);
}

void launch_fit(const ImgDesc* d_descs, int nimg, int max_sort_tiles, long long max_nodes, int max_chunks,
                cudaStream_t st, bool any_hist) {
  launch_fit_sort(d_descs, nimg, max_sort_tiles, st, any_hist);
  launch_fit_bins(d_descs, nimg, max_nodes, max_chunks, st);
}

// ---------------------------------------------------------------------------
// Tile-sharded fit: an owner rank's received samples, one chunk per source
// rank ([3][m] f64 S*, then [3][m] u8 M, each chunk sorted by exponent), are
// regrouped bin-major with the sources in rank order inside a bin -- which is
// raster order, since the bands are contiguous row ranges.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fit_regroup(const ImgDesc* __restrict__ descs, RegroupTab rt) {
  const ImgDesc& d = descs[0];
  const long long M = d.fit_m;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < rt.total;
       i += (long long)gridDim.x * blockDim.x) {
    int r = 0;  // source chunk: cumulative sample counts
    long long before = 0;
    while (r + 1 < rt.nsrc && before + rt.src_m[r] <= i) before += rt.src_m[r++];
    const long long j = i - before, m = rt.src_m[r];
    const unsigned* bo = rt.src_bin_off + (long long)r * 257;
    int lo = 0, hi = 256;  // bin e with bo[e] <= j < bo[e+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bo[mid] <= j) lo = mid; else hi = mid;
    }
    const long long dst = (long long)rt.dst_bin_off[r * 256 + lo] + (j - bo[lo]);
    const uint8_t* chunk = rt.recv + rt.src_off[r];
    const double* x = reinterpret_cast<const double*>(chunk);
    const uint8_t* y = chunk + 24 * m;
#pragma unroll
    for (int c = 0; c < 3; c++) {
      d.xs[c * M + dst] = x[c * m + j];
      d.ys[c * M + dst] = y[c * m + j];
    }
  }
}

void launch_fit_regroup(const ImgDesc* d_desc, const RegroupTab& rt, cudaStream_t st) {
  if (rt.total <= 0) return;
  long long blocks = (rt.total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_fit_regroup<<<(unsigned)blocks, 256, 0, st>>>(d_desc, rt);
}

void upload_fit_constants() { upload_pw_table(); }

}  // namespace hdll
