// tonemap.cu -- RGBE unpack + global Reinhard statistics pass.
//
// Reference: tonemap.py:74-110 (luminance, log-average, white point) over
// rgbe.py:70-90 (rgbe_to_float).  Pass A here computes per pixel
// Lw = (0.2126 R + 0.7152 G) + 0.0722 B and log(eps + Lw) in fp64, plus the
// image max of Lw; the log-average is numpy's pairwise mean of those logs
// (pairwise.cuh).  The per-pixel mapping pass B is fused into the base-layer
// kernel (base.cu), which is where the SDR is consumed.
#include "encoder.cuh"
#include "pairwise.cuh"

namespace hdll {

// rgbe_to_float for one component: ldexp((m + 0.5) / 256, e - 128), exact.
__device__ __forceinline__ double rgbe_comp(unsigned m, double scale) { return ((double)m + 0.5) * scale; }

// 2^(e-136) as a double (e in [0, 255] gives a normal number)
__device__ __forceinline__ double rgbe_scale(unsigned e) {
  return __longlong_as_double((long long)((int)e - 136 + 1023) << 52);
}

__device__ __forceinline__ void rgbe_to_rgb(uint32_t q, double* r, double* g, double* b) {
  if (q == 0u) {
    *r = *g = *b = 0.0;
    return;
  }
  double sc = rgbe_scale(q >> 24);
  *r = rgbe_comp(q & 0xFF, sc);
  *g = rgbe_comp((q >> 8) & 0xFF, sc);
  *b = rgbe_comp((q >> 16) & 0xFF, sc);
}

// luminance, tonemap.py:74-77 (Rec.709 weights, left-to-right, no FMA)
__device__ __forceinline__ double luminance(double r, double g, double b) {
  return 0.2126 * r + 0.7152 * g + 0.0722 * b;
}

// Pass A over full-image pixels [px0, px1): 4 pixels per thread (one 128-bit
// load when aligned).  logv and rgbe are indexed in desc pixels (p - pix_base).
__global__ void __launch_bounds__(256) k_lum_log(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const long long q0 = d.px0 - d.pix_base, q1 = d.px1 - d.pix_base;  // desc pixels
  const long long lead = (4 - (q0 & 3)) & 3;                         // pixels before the first aligned quad
  const long long nq = (q1 - q0 - lead + 3) / 4;
  double mx = 0.0;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(d.rgbe);
  for (long long qi = (long long)blockIdx.x * blockDim.x + threadIdx.x; qi < nq + 1;
       qi += (long long)gridDim.x * blockDim.x) {
    long long p0;
    int cnt;
    uint32_t qs[4];
    if (qi == nq) {  // the unaligned lead pixels
      p0 = q0;
      cnt = (int)min(lead, q1 - q0);
      for (int k = 0; k < cnt; k++) qs[k] = src[p0 + k];
    } else {
      p0 = q0 + lead + qi * 4;
      cnt = (int)min(4LL, q1 - p0);
      if (cnt == 4) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(src + p0));
        qs[0] = v.x, qs[1] = v.y, qs[2] = v.z, qs[3] = v.w;
      } else {
        for (int k = 0; k < cnt; k++) qs[k] = src[p0 + k];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (k >= cnt) break;
      double r, g, b;
      rgbe_to_rgb(qs[k], &r, &g, &b);
      double lw = luminance(r, g, b);
      mx = fmax(mx, lw);
      d.logv[p0 + k] = log(d.epsilon + lw);
    }
  }
  // block max -> one atomic (Lw >= 0 so the bit pattern orders like the value)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = wmax[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) m = fmax(m, wmax[i]);
    atomicMax(d.maxlw, (unsigned long long)__double_as_longlong(m));
  }
}

struct PtrAcc {  // full-image index -> desc array
  const double* p;
  long long base;
  __device__ double operator()(long long i) const { return p[i - base]; }
};

// Pairwise-sum depth-L nodes [node0, node1) of every image's log array.
__global__ void __launch_bounds__(128) k_tm_nodes(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  long long idx = d.node0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d.node1) return;
  long long off, sz;
  pairwise_node(d.full_n, d.tm_level, idx, &off, &sz);
  d.tm_nodes[idx] = pairwise_seq(PtrAcc{d.logv, d.pix_base}, off, sz);
}

// Combine the nodes, then the scalar tail of tone_map (tonemap.py:97-104).
__global__ void __launch_bounds__(256) k_tm_scalars(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.x];
  __shared__ double sm[256];
  double sum = tree_reduce_block(d.tm_nodes, d.tm_level, sm);
  if (threadIdx.x == 0) {
    double total = 0.0 + sum;                       // reduction initial value 0.0
    double mean = total / (double)d.full_n;         // np.mean: sum / count
    double log_avg = exp(mean);
    double maxlw = __longlong_as_double((long long)*d.maxlw);
    double white = d.white_point > 0 ? d.white_point : d.key * maxlw / log_avg;  // == scaled.max()
    d.scalars[0] = total;
    d.scalars[1] = log_avg;
    d.scalars[2] = white;
    d.scalars[3] = (maxlw > 0.0) ? 0.0 : 1.0;      // all-black input (tonemap.py:97-99)
  }
}

void launch_tonemap_partial(const ImgDesc* d_descs, int nimg, long long max_n, int max_level, cudaStream_t st) {
  long long nq = (max_n + 3) / 4 + 1;
  int gx = (int)((nq + 255) / 256);
  if (gx > 148 * 8) gx = 148 * 8;
  if (gx < 1) gx = 1;
  k_lum_log<<<dim3(gx, nimg), 256, 0, st>>>(d_descs);
  long long nn = 1LL << max_level;
  k_tm_nodes<<<dim3((unsigned)((nn + 127) / 128), nimg), 128, 0, st>>>(d_descs);
}

void launch_tonemap_scalars(const ImgDesc* d_descs, int nimg, cudaStream_t st) {
  k_tm_scalars<<<nimg, 256, 0, st>>>(d_descs);
}

void launch_tonemap_stats(const ImgDesc* d_descs, int nimg, long long max_n, int max_level, cudaStream_t st) {
  launch_tonemap_partial(d_descs, nimg, max_n, max_level, st);
  launch_tonemap_scalars(d_descs, nimg, st);
}

}  // namespace hdll
