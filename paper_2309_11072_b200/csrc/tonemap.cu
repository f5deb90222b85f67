// tonemap.cu -- RGBE unpack + global Reinhard statistics pass.
//
// Reference: tonemap.py:74-110 (luminance, log-average, white point) over
// rgbe.py:70-90 (rgbe_to_float).  Pass A here computes per pixel
// Lw = (0.2126 R + 0.7152 G) + 0.0722 B and log(eps + Lw) in fp64 inside
// numpy's pairwise mean of those logs (pairwise.cuh), plus the image max of
// Lw.  The per-pixel mapping pass B is fused into the base-layer
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

// Pass A, fused: one warp per depth-L node of numpy's pairwise tree over the
// full image (nodes [node0, node1) of this desc).  The node's elements
// log(eps + Lw) are computed where the tree reads them (warp_pairwise reads
// every element exactly once), so the logs never touch memory; the same pass
// takes the max of Lw.  rgbe is indexed in desc pixels (p - pix_base).
struct LogLwAcc {
  const uint32_t* px;
  long long base;
  double eps;
  double* mx;  // the calling lane's running max of Lw
  __device__ __forceinline__ double operator()(long long i) const {
    double r, g, b;
    rgbe_to_rgb(__ldg(px + (i - base)), &r, &g, &b);
    const double lw = luminance(r, g, b);
    *mx = fmax(*mx, lw);
    return log(eps + lw);
  }
};

__global__ void __launch_bounds__(128) k_tm_nodes(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  __shared__ PwScratch pw[4];
  const int warp = threadIdx.x >> 5;
  const long long idx = d.node0 + (long long)blockIdx.x * 4 + warp;
  double mx = 0.0;
  if (idx < d.node1) {
    long long off, sz;
    pairwise_node(d.full_n, d.tm_level, idx, &off, &sz);
    const double r = warp_pairwise<LogLwAcc, false>(
        LogLwAcc{reinterpret_cast<const uint32_t*>(d.rgbe), d.pix_base, d.epsilon, &mx}, off, sz, pw[warp]);
    if ((threadIdx.x & 31) == 0) d.tm_nodes[idx] = r;
  }
  // block max -> one atomic (Lw >= 0 so the bit pattern orders like the value)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double wmax[4];
  if ((threadIdx.x & 31) == 0) wmax[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double m = fmax(fmax(wmax[0], wmax[1]), fmax(wmax[2], wmax[3]));
    if (m > 0.0) atomicMax(d.maxlw, (unsigned long long)__double_as_longlong(m));
  }
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
  (void)max_n;
  const long long nn = 1LL << max_level;
  k_tm_nodes<<<dim3((unsigned)((nn + 3) / 4), nimg), 128, 0, st>>>(d_descs);
}

void launch_tonemap_scalars(const ImgDesc* d_descs, int nimg, cudaStream_t st) {
  k_tm_scalars<<<nimg, 256, 0, st>>>(d_descs);
}

void launch_tonemap_stats(const ImgDesc* d_descs, int nimg, long long max_n, int max_level, cudaStream_t st) {
  launch_tonemap_partial(d_descs, nimg, max_n, max_level, st);
  launch_tonemap_scalars(d_descs, nimg, st);
}

void upload_tonemap_constants() { upload_pw_table(); }

}  // namespace hdll
