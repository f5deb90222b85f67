// prefilter.cu -- Gaussian prefilter S -> S* (estimator.py:130-142).
//
// scipy.ndimage.correlate1d with a symmetric odd kernel and mode="reflect",
// axis 0 then axis 1 (scipy/ndimage/src/ni_filters.c NI_Correlate1D,
// symmetric branch):
//   out[i] = x[i] * w[r];  for jj = -r .. -1: out[i] += (x[i+jj] + x[i-jj]) * w[r+jj]
// reflect index: m = i mod 2n; m >= n -> 2n - 1 - m (lines shorter than r
// reflect repeatedly).  Verified in oracle/hdll_oracle.c ho_prefilter.
//
// Two passes: vertical (u8 S -> f64 scratch, coalesced along x) and horizontal
// (f64 scratch -> f64 S*, the row staged in shared memory with its reflected
// halo).  Taps come from the host (numpy gaussian_kernel) via d.taps.
#include "encoder.cuh"

namespace hdll {

__device__ __forceinline__ int reflect_idx(long long i, long long n) {
  long long m = i % (2 * n);
  if (m < 0) m += 2 * n;
  if (m >= n) m = 2 * n - 1 - m;
  return (int)m;
}

// grid: (ceil(w/128), h, nimg*3) ; one thread per output pixel
__global__ void __launch_bounds__(128) k_prefilter_v(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.z / 3];
  const int c = blockIdx.z % 3;
  if (!d.slrme || d.sigma_milli == 0) return;
  const int y = blockIdx.y, x = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= d.h || x >= d.w) return;
  const uint8_t* S = d.s_planes + (long long)c * d.n;
  const int r = d.radius;
  const double* fw = d.taps + r;
  double o = (double)S[(long long)y * d.w + x] * fw[0];
  for (int jj = -r; jj < 0; jj++) {
    double lo = S[(long long)reflect_idx(y + jj, d.h) * d.w + x];
    double hi = S[(long long)reflect_idx(y - jj, d.h) * d.w + x];
    o += (lo + hi) * fw[jj];
  }
  d.sstar_tmp[(long long)c * d.n + (long long)y * d.w + x] = o;
}

// grid: (ceil(w/256), h, nimg*3); the row segment plus reflected halo in smem
__global__ void __launch_bounds__(256) k_prefilter_h(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.z / 3];
  const int c = blockIdx.z % 3;
  if (!d.slrme || d.sigma_milli == 0) return;
  const int y = blockIdx.y;
  if (y >= d.h) return;
  const int x0 = blockIdx.x * blockDim.x;
  if (x0 >= d.w) return;
  const int r = d.radius;
  const double* fw = d.taps + r;
  const double* row = d.sstar_tmp + (long long)c * d.n + (long long)y * d.w;
  extern __shared__ double seg[];  // blockDim.x + 2r values: logical x in [x0 - r, x0 + blockDim.x + r)
  const int span = blockDim.x + 2 * r;
  for (int i = threadIdx.x; i < span; i += blockDim.x) seg[i] = row[reflect_idx((long long)x0 - r + i, d.w)];
  __syncthreads();
  const int x = x0 + threadIdx.x;
  if (x >= d.w) return;
  const double* s = seg + r + threadIdx.x;
  double o = s[0] * fw[0];
  for (int jj = -r; jj < 0; jj++) o += (s[jj] + s[-jj]) * fw[jj];
  d.sstar[(long long)c * d.n + (long long)y * d.w + x] = o;
}

// Fused single pass for radius <= kFusedMaxR: one CTA = kTH x kTW outputs of one
// channel; the u8 input tile with its reflected halo and the vertical-pass
// rows stay in shared memory; only S* is written.
constexpr int kTH = 32, kTW = 64, kFusedMaxR = 16;

struct PfSmem {
  uint8_t in[(kTH + 2 * kFusedMaxR) * (kTW + 2 * kFusedMaxR)];
  double tmp[kTH * (kTW + 2 * kFusedMaxR)];
  double fw_s[2 * kFusedMaxR + 1];
  int gys[kTH + 2 * kFusedMaxR], gxs[kTW + 2 * kFusedMaxR];
};

template <int R>  // R > 0: compile-time radius; R == 0: runtime d.radius
__device__ __forceinline__ void prefilter_tile(const ImgDesc& d, int c, int y0, int x0, PfSmem& sm) {
  const int r = R > 0 ? R : d.radius;
  const int IW = kTW + 2 * r, IH = kTH + 2 * r;
  uint8_t* in = sm.in;
  double* tmp = sm.tmp;
  double* fw_s = sm.fw_s;
  int* gys = sm.gys;
  int* gxs = sm.gxs;
  const uint8_t* S = d.s_planes + (long long)c * d.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 2 * r + 1; i += blockDim.x) fw_s[i] = d.taps[i];
  for (int i = threadIdx.x; i < IH; i += blockDim.x) gys[i] = reflect_idx((long long)y0 - r + i, d.h);
  for (int i = threadIdx.x; i < IW; i += blockDim.x) gxs[i] = reflect_idx((long long)x0 - r + i, d.w);
  __syncthreads();
  for (int ry = warp; ry < IH; ry += nwarp) {
    const uint8_t* srow = S + (long long)gys[ry] * d.w;
    for (int rx = lane; rx < IW; rx += 32) in[ry * IW + rx] = srow[gxs[rx]];
  }
  __syncthreads();
  const double* fw = fw_s + r;
  // vertical pass (axis 0) for every staged column
  for (int oy = warp; oy < kTH; oy += nwarp) {
    for (int col = lane; col < IW; col += 32) {
      const uint8_t* cp = in + (oy + r) * IW + col;
      double o = (double)cp[0] * fw[0];
#pragma unroll
      for (int jj = -r; jj < 0; jj++) o += ((double)cp[jj * IW] + (double)cp[-jj * IW]) * fw[jj];
      tmp[oy * IW + col] = o;
    }
  }
  __syncthreads();
  // horizontal pass (axis 1)
  for (int oy = warp; oy < kTH; oy += nwarp) {
    const int y = y0 + oy;
    if (y >= d.h) break;
    for (int ox = lane; ox < kTW; ox += 32) {
      const int x = x0 + ox;
      if (x >= d.w) break;
      const double* rp = tmp + oy * IW + ox + r;
      double o = rp[0] * fw[0];
#pragma unroll
      for (int jj = -r; jj < 0; jj++) o += (rp[jj] + rp[-jj]) * fw[jj];
      d.sstar[(long long)c * d.n + (long long)y * d.w + x] = o;
    }
  }
}

__global__ void __launch_bounds__(256) k_prefilter_fused(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.z / 3];
  const int c = blockIdx.z % 3;
  if (!d.slrme || d.sigma_milli == 0 || d.radius > kFusedMaxR || d.radius == 3) return;
  const int tiles_x = (d.w + kTW - 1) / kTW;
  const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
  const int y0 = ty * kTH, x0 = tx * kTW;
  if (y0 >= d.h) return;
  __shared__ PfSmem sm;
  prefilter_tile<0>(d, c, y0, x0, sm);  // radius 3 (sigma 1.0, the default) runs in k_prefilter_cols
}

// Column kernel for a compile-time radius R (the default sigma = 1 has R = 3):
// a CTA of 256 threads owns 256 - 2R output columns x kCR output rows of one
// channel.  Vertical pass: thread = staged column, a (2R + 1)-sample window
// slides down it in registers (coalesced u8 row loads).  Horizontal pass:
// thread = output column, reading the vertical results of its row from
// shared memory.  Same operation order as scipy's symmetric branch.
constexpr int kCR = 16;

template <int R>
__global__ void __launch_bounds__(256) k_prefilter_cols(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.z / 3];
  const int c = blockIdx.z % 3;
  if (!d.slrme || d.sigma_milli == 0 || d.radius != R) return;
  constexpr int kOut = 256 - 2 * R;
  const int tiles_x = (d.w + kOut - 1) / kOut;
  const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
  const int y0 = ty * kCR, x0 = tx * kOut;
  if (y0 >= d.h) return;
  __shared__ double vt[kCR][256 + 1];
  const int t = threadIdx.x;
  double fw[R + 1];  // fw[j] = taps[R - j]: centre, then outward
#pragma unroll
  for (int j = 0; j <= R; j++) fw[j] = d.taps[R - j];
  const uint8_t* S = d.s_planes + (long long)c * d.n;
  const int gx = reflect_idx((long long)x0 - R + t, d.w);
  // vertical pass over rows y0 .. y0 + kCR - 1 of column gx; away from the top
  // and bottom edges the rows are consecutive (no reflection arithmetic)
  const bool inner = y0 >= R && y0 + kCR + R <= d.h;
  const uint8_t* col = S + gx;
  const long long W = d.w;
  const uint8_t* rp = col + (inner ? (long long)(y0 - R) * W : 0);
  // all kCR + 2R input bytes of the column in flight at once (the pass is
  // otherwise bound by one dependent load latency per output row)
  uint8_t colv[kCR + 2 * R];
  if (inner) {
#pragma unroll
    for (int i = 0; i < kCR + 2 * R; i++) colv[i] = __ldg(rp + (long long)i * W);
  } else {
#pragma unroll
    for (int i = 0; i < kCR + 2 * R; i++)
      colv[i] = __ldg(col + (long long)reflect_idx((long long)y0 - R + i, d.h) * W);
  }
  double win[2 * R + 1];
#pragma unroll
  for (int i = 0; i < 2 * R; i++) win[i + 1] = (double)colv[i];
#pragma unroll
  for (int oy = 0; oy < kCR; oy++) {
#pragma unroll
    for (int i = 0; i < 2 * R; i++) win[i] = win[i + 1];
    win[2 * R] = (double)colv[oy + 2 * R];
    double o = win[R] * fw[0];
#pragma unroll
    for (int j = R; j >= 1; j--) o += (win[R - j] + win[R + j]) * fw[j];
    vt[oy][t] = o;
  }
  __syncthreads();
  // horizontal pass
  const int x = x0 + t - R;
  if (t < R || t >= 256 - R || x >= d.w) return;
  double* out = d.sstar + (long long)c * d.n + (long long)y0 * W + x;
  const int rows = min(kCR, d.h - y0);
#pragma unroll 4
  for (int oy = 0; oy < rows; oy++) {
    double o = vt[oy][t] * fw[0];
#pragma unroll
    for (int j = R; j >= 1; j--) o += (vt[oy][t - j] + vt[oy][t + j]) * fw[j];
    *out = o;
    out += W;
  }
}

void launch_prefilter(const ImgDesc* d_descs, int nimg, int max_w, int max_h, int max_radius, cudaStream_t st,
                      bool any_non3) {
  if (max_radius >= 3) {  // the images of radius 3 (sigma 1, the default); the others return at once
    const int tiles = ((max_w + 249) / 250) * ((max_h + kCR - 1) / kCR);
    k_prefilter_cols<3><<<dim3(tiles, 1, nimg * 3), 256, 0, st>>>(d_descs);
  }
  if (!any_non3) return;
  if (max_radius <= kFusedMaxR) {  // (images of other radii; radius-3 ones return at once)
    const int tiles = ((max_w + kTW - 1) / kTW) * ((max_h + kTH - 1) / kTH);
    k_prefilter_fused<<<dim3(tiles, 1, nimg * 3), 256, 0, st>>>(d_descs);
    return;
  }
  k_prefilter_v<<<dim3((max_w + 127) / 128, max_h, nimg * 3), 128, 0, st>>>(d_descs);
  size_t smem = sizeof(double) * (256 + 2 * (size_t)max_radius);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_prefilter_h, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_prefilter_h<<<dim3((max_w + 255) / 256, max_h, nimg * 3), 256, smem, st>>>(d_descs);
}

}  // namespace hdll
