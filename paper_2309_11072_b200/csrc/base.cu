// base.cu -- tone-map pass B + the base-layer 8x8 DCT round trip, fused.
//
// Reference chain (container.py:167-172):
//   tone_map mapping pass          tonemap.py:100-110, srgb_quantize :113-118
//   _BlockDctCoder.encode          codec_core.py:430-453
//     np.pad edge / _rgb_to_ycc    :432-436, :391-403
//     dct_blocks                   _kernels.py:381-400
//     round_half_away(coef / qt)   :447, zigzag :448
//   _reconstruct (== lossy_decode) codec_core.py:478-489, idct_blocks _kernels.py:403-422,
//                                  _ycc_to_rgb :406-411
// The reference obtains S by entropy-decoding its own payload (container.py:172);
// that decode reproduces exactly the zz it just coded, so S is reconstructed here
// straight from zz -- the entropy coder (entropy.cu) runs
// separately on the same zz.
//
// One CTA = 8 pixel rows x 128 columns (16 blocks) of one image, 128 threads.
// All block transforms stay in shared memory; fp64 with no contraction and the
// reference's summation order (s = 0.0; s += C * x for t = 0..7).
#include <algorithm>

#include "encoder.cuh"

namespace hdll {

// DCT_MATRIX, _kernels.py:23-43 (row u, column t), compile-time constants so the
// fully unrolled transforms take them as instruction operands
__device__ constexpr double kDctM[64] = {
      0.35355339059327373, 0.35355339059327373, 0.35355339059327373, 0.35355339059327373,
      0.35355339059327373, 0.35355339059327373, 0.35355339059327373, 0.35355339059327373,
      0.4903926402016152,  0.4157348061512726,  0.27778511650980114, 0.09754516100806417,
      -0.0975451610080641, -0.277785116509801,  -0.4157348061512727, -0.4903926402016152,
      0.46193976625564337, 0.19134171618254492, -0.19134171618254486, -0.46193976625564337,
      -0.4619397662556434, -0.19134171618254517, 0.191341716182545,   0.46193976625564326,
      0.4157348061512726,  -0.0975451610080641, -0.4903926402016152, -0.2777851165098011,
      0.2777851165098009,  0.4903926402016152,  0.09754516100806439, -0.41573480615127256,
      0.3535533905932738,  -0.35355339059327373, -0.35355339059327384, 0.3535533905932737,
      0.35355339059327384, -0.35355339059327334, -0.35355339059327356, 0.3535533905932733,
      0.27778511650980114, -0.4903926402016152, 0.09754516100806415, 0.41573480615127273,
      -0.41573480615127256, -0.09754516100806401, 0.4903926402016153, -0.27778511650980076,
      0.19134171618254492, -0.4619397662556434, 0.46193976625564326, -0.19134171618254495,
      -0.19134171618254528, 0.46193976625564337, -0.4619397662556432, 0.19134171618254478,
      0.09754516100806417, -0.2777851165098011, 0.41573480615127273, -0.4903926402016153,
      0.4903926402016152,  -0.4157348061512725, 0.27778511650980076, -0.09754516100806429};
__constant__ int c_zigzag[64];  // ZIGZAG, codec_core.py:364-372

constexpr int kTileBlocks = 16;
constexpr int kTileCols = kTileBlocks * 8;  // 128
constexpr int kRowStride = kTileCols + 1;   // doubles; padding against bank conflicts


__device__ __forceinline__ double rgbe_scale_b(unsigned e) {
  return __longlong_as_double((long long)((int)e - 136 + 1023) << 52);
}

// srgb_quantize(pow(m, g)) = round_half_away(255 * clip(m^g, 0, 1)) for m >= 0.
// The quantised byte only depends on which side of k + 0.5 the product lies,
// so it is first evaluated in fp32 (log2f 1 ulp, exp2f 2 ulp, m rounded to fp32:
// |err(255 m^g)| < 1e-3 for g <= 32, normal fp32 m) and accepted when 255 m^g + 0.5 is more than kAmb away
// from an integer; otherwise the fp64 pow decides (as numpy's does; numpy's
// own power is SVML, not correctly rounded).
constexpr float kAmb = 2e-3f;

__device__ __noinline__ uint8_t quantize_pow_exact(double m, double g) {
  double v = pow(m, g);
  return (uint8_t)rha(255.0 * clampd(v, 0.0, 1.0));
}

// For 1 / gamma <= 4 the fp32 pass uses the MUFU approximations (lg2 / ex2
// .approx: ~2^-22 relative): |err(255 m^g)| stays below 4e-4, well inside kAmb.
constexpr float kApproxMaxG = 4.0f;
// The fp32 pass at all: |err(255 m^g)| ~ 255 g 2^-24 (m's rounding) + 2e-4 stays
// below kAmb / 2 up to g = 32; larger 1 / gamma always takes the fp64 pow.
constexpr float kFastMaxG = 32.0f;

__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 1 / x from the MUFU approximation and one Newton step (relative error
// ~2^-40; x normal and finite)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// the byte, or -1 when the fp32 value is too close to a rounding boundary
__device__ __forceinline__ int quantize_pow_fast(double m, float g32, bool approx) {
  if (m >= 1.0) return 255;  // m^g >= 1 clips to 1
  if (m <= 0.0) return 0;
  const float mf = __double2float_rn(m);
  // Outside the certified range the fp64 pow decides: an m below FLT_MIN has
  // no normal fp32 image (lg2.approx.ftz flushes it, a subnormal loses bits,
  // and a zero would give byte 0 where m^g can be far from 0 for small g);
  // rounding m to fp32 contributes ~255 g 2^-24 to 255 m^g, inside kAmb only
  // for g <= kFastMaxG.
  if (!(mf >= 1.17549435e-38f) || g32 > kFastMaxG) return -1;
  const float y = 255.0f * (approx ? ex2_approx(g32 * lg2_approx(mf)) : exp2f(g32 * log2f(mf)));
  const float yf = y + 0.5f;
  const float fl = floorf(yf), fr = yf - fl;
  if (fr > kAmb && fr < 1.0f - kAmb) return (int)fl;
  return -1;
}

// tone_map pass B for one pixel -> 3 SDR bytes (fp64 chain of the reference,
// tonemap.py:102-110; the gamma step through quantize_pow_fast, and with
// `exact` the fp64 pow for whatever the fast pass cannot certify).  Returns
// false when a byte is undecided (exact == false only).
struct TmoConst {
  float g32;     // 1 / gamma
  bool approx;   // g32 <= kApproxMaxG
  double inv_la, inv_w2;  // refined reciprocals of log_avg and white^2 (fast pass)
};

__device__ __forceinline__ bool sdr_pixel(const ImgDesc& d, uint32_t q, double log_avg, double white,
                                          const TmoConst& tc, bool allzero, uint8_t* out3, bool exact) {
  if (allzero || q == 0u) {
    out3[0] = out3[1] = out3[2] = 0;
    return true;
  }
  const double sc = rgbe_scale_b(q >> 24);
  double f[3];
  f[0] = ((double)(q & 0xFF) + 0.5) * sc;
  f[1] = ((double)((q >> 8) & 0xFF) + 0.5) * sc;
  f[2] = ((double)((q >> 16) & 0xFF) + 0.5) * sc;
  const double lw = 0.2126 * f[0] + 0.7152 * f[1] + 0.0722 * f[2];
  double ratio;
  if (exact) {  // the reference's fp64 chain, every division correctly rounded
    const double scaled = d.key * lw / log_avg;
    const double disp = scaled * (1.0 + scaled / (white * white)) / (1.0 + scaled);
    ratio = lw > 0 ? disp / lw : 0.0;
  } else {  // divisions as refined reciprocals (~2^-40): far inside the kAmb window
    const double scaled = d.key * lw * tc.inv_la;
    const double disp = scaled * (1.0 + scaled * tc.inv_w2) * rcp_nr(1.0 + scaled);
    ratio = lw > 0 ? disp * rcp_nr(lw) : 0.0;
  }
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const double m = fmax(f[c] * ratio, 0.0);
    int v = quantize_pow_fast(m, tc.g32, tc.approx);
    if (v < 0) {
      if (exact) v = quantize_pow_exact(m, d.inv_gamma);
      else ok = false;
    }
    out3[c] = (uint8_t)v;
  }
  return ok;
}

// Pass 1, per pixel: tone-map pass B (or the given SDR in the lossy-coder
// plugin mode) and _rgb_to_ycc with rounding and clamping (codec_core.py:391-403),
// stored as bytes (Y in [0, 255], Cb / Cr in [-128, 127]).  Four pixels per
// thread; the transform kernel below reads them back per 8x8 block.  Split from
// the transforms so each runs at its own register budget.

__device__ __forceinline__ void ycc_bytes(const uint8_t* s3, uint8_t* y, int8_t* cb, int8_t* cr) {
  const double r = s3[0], g = s3[1], b = s3[2];
  const double Y = 0.299 * r + 0.587 * g + 0.114 * b;
  const double u = -0.168736 * r - 0.331264 * g + 0.5 * b;
  const double v = 0.5 * r - 0.418688 * g - 0.081312 * b;
  *y = (uint8_t)min(max(rha_int(Y), 0), 255);
  *cb = (int8_t)min(max(rha_int(u), -128), 127);
  *cr = (int8_t)min(max(rha_int(v), -128), 127);
}

// _rgb_to_ycc of one pixel as Y | Cb << 8 | Cr << 16.  (An exact-integer form
// with a tie fallback was measured slower: the fp64 pipe has room here, the
// integer pipes do not.)
__device__ __forceinline__ uint32_t ycc_word(const uint8_t* s3) {
  uint8_t Y;
  int8_t Cb, Cr;
  ycc_bytes(s3, &Y, &Cb, &Cr);
  return (uint32_t)Y | ((uint32_t)(uint8_t)Cb << 8) | ((uint32_t)(uint8_t)Cr << 16);
}

__global__ void __launch_bounds__(256) k_sdr_ycc(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const double log_avg = d.sdr_in ? 1.0 : d.scalars[1], white = d.sdr_in ? 1.0 : d.scalars[2];
  const bool allzero = d.sdr_in ? false : d.scalars[3] != 0.0;
  TmoConst tc;
  tc.g32 = (float)d.inv_gamma;
  tc.approx = tc.g32 <= kApproxMaxG;
  tc.inv_la = rcp_nr(log_avg);
  tc.inv_w2 = rcp_nr(white * white);
  const long long nq = (d.n + 3) / 4;
  uint8_t* Yp = d.ycc;
  uint8_t* Cb = d.ycc + d.n;
  uint8_t* Cr = d.ycc + 2 * d.n;
  const bool aligned = (d.n & 3) == 0;  // the planes' 4-pixel groups are 4-byte aligned
  // The fit's exponent histogram per 1024-pixel sort tile (fit.cu k_sort_hist)
  // rides along: one pass of this grid-stride loop is exactly one sort tile.
  // Two buffers, one barrier per pass: a thread clears its entry of the next
  // pass's buffer before the barrier that ends this pass's counting.
  __shared__ unsigned hist[2][256];
  const bool fuse_hist = d.hist_fused != 0;
  static_assert(kSortTile == 4 * 256, "one k_sdr_ycc block iteration covers one sort tile");
  if (fuse_hist) {
    hist[0][threadIdx.x] = 0;
    __syncthreads();
  }
  int buf = 0;
  for (long long qb = (long long)blockIdx.x * blockDim.x; qb < nq; qb += (long long)gridDim.x * blockDim.x) {
    const long long qi = qb + threadIdx.x;
    if (fuse_hist) hist[buf ^ 1][threadIdx.x] = 0;
    const long long p0 = qi * 4;
    const int cnt = qi < nq ? (int)min(4LL, d.n - p0) : 0;
    uint32_t qs[4] = {0u, 0u, 0u, 0u};
    if (!d.sdr_in && cnt > 0) {
      if (cnt == 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(d.rgbe) + qi);
        qs[0] = v.x, qs[1] = v.y, qs[2] = v.z, qs[3] = v.w;
      } else {
        for (int k = 0; k < cnt; k++) qs[k] = reinterpret_cast<const uint32_t*>(d.rgbe)[p0 + k];
      }
    }
    uint32_t yw = 0, cbw = 0, crw = 0;  // the 4 pixels' bytes (a deferred pixel's are written by k_sdr_fix)
    // The four pixels' fast passes as one straight-line block: independent
    // fp64 chains the scheduler interleaves (the kernel's top stall is the
    // fixed-latency dependency wait; A/B config 1: base 4.05 -> 3.99 ms).  A
    // pixel past cnt has q = 0 and costs a select.  Then the rare deferrals
    // and the packing.  (The SDR-input plugin mode and the trace keep the
    // per-pixel loop below.)
    if (!d.sdr_in && !d.want_trace) {
      uint8_t s4[4][3];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) ok[k] = sdr_pixel(d, qs[k], log_avg, white, tc, allzero, s4[k], false);
      uint32_t w4[4];
#pragma unroll
      for (int k = 0; k < 4; k++) w4[k] = ycc_word(s4[k]);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (k >= cnt) break;
        if (!ok[k]) {
          const unsigned slot = atomicAdd(d.amb, 1u);
          if (slot < d.amb_cap) {
            d.amb_list[slot] = (unsigned)(p0 + k);
            continue;
          }
          sdr_pixel(d, qs[k], log_avg, white, tc, allzero, s4[k], true);  // list full: here
          w4[k] = ycc_word(s4[k]);
        }
        yw |= (w4[k] & 0xFFu) << (8 * k);
        cbw |= ((w4[k] >> 8) & 0xFFu) << (8 * k);
        crw |= ((w4[k] >> 16) & 0xFFu) << (8 * k);
      }
    } else
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (k >= cnt) break;
      const long long p = p0 + k;
      uint8_t s3[3];
      bool have = true;
      if (d.sdr_in) {
        s3[0] = d.sdr_in[3 * p], s3[1] = d.sdr_in[3 * p + 1], s3[2] = d.sdr_in[3 * p + 2];
      } else if (!sdr_pixel(d, qs[k], log_avg, white, tc, allzero, s3, false)) {
        // a byte the fp32 pass cannot certify (~0.3 % of samples): the pixel
        // goes to k_sdr_fix instead of holding its warp through an fp64 pow
        const unsigned slot = atomicAdd(d.amb, 1u);
        if (slot < d.amb_cap) {
          d.amb_list[slot] = (unsigned)p;
          have = false;
        } else {
          sdr_pixel(d, qs[k], log_avg, white, tc, allzero, s3, true);  // list full: here
        }
      }
      if (have) {
        if (d.want_trace && !d.sdr_in) {
          d.sdr[3 * p] = s3[0];
          d.sdr[3 * p + 1] = s3[1];
          d.sdr[3 * p + 2] = s3[2];
        }
        const uint32_t w = ycc_word(s3);
        yw |= (w & 0xFFu) << (8 * k);
        cbw |= ((w >> 8) & 0xFFu) << (8 * k);
        crw |= ((w >> 16) & 0xFFu) << (8 * k);
      }
    }
    if (cnt == 4 && aligned) {
      reinterpret_cast<uint32_t*>(Yp)[qi] = yw;
      reinterpret_cast<uint32_t*>(Cb)[qi] = cbw;
      reinterpret_cast<uint32_t*>(Cr)[qi] = crw;
    } else {
      for (int k = 0; k < cnt; k++) {
        Yp[p0 + k] = (uint8_t)(yw >> (8 * k));
        Cb[p0 + k] = (uint8_t)(cbw >> (8 * k));
        Cr[p0 + k] = (uint8_t)(crw >> (8 * k));
      }
    }
    if (fuse_hist) {
      for (int k = 0; k < cnt; k++) atomicAdd(&hist[buf][qs[k] >> 24], 1u);
      __syncthreads();
      const unsigned hc = hist[buf][threadIdx.x];
      d.tile_hist[(long long)threadIdx.x * d.sort_tiles + qb / 256] = hc;
      if (hc) atomicAdd(&d.bin_count[threadIdx.x], hc);
      buf ^= 1;
    }
  }
}

// the deferred pixels of k_sdr_ycc, with the fp64 pow where needed
__global__ void __launch_bounds__(256) k_sdr_fix(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  if (d.sdr_in) return;
  const unsigned cnt = min(*d.amb, d.amb_cap);
  TmoConst tc;
  tc.g32 = (float)d.inv_gamma;
  tc.approx = tc.g32 <= kApproxMaxG;
  const double log_avg = d.scalars[1], white = d.scalars[2];
  tc.inv_la = rcp_nr(log_avg);
  tc.inv_w2 = rcp_nr(white * white);
  const bool allzero = d.scalars[3] != 0.0;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const long long p = d.amb_list[i];
    uint8_t s3[3];
    sdr_pixel(d, reinterpret_cast<const uint32_t*>(d.rgbe)[p], log_avg, white, tc, allzero, s3, true);
    if (d.want_trace) {
      d.sdr[3 * p] = s3[0];
      d.sdr[3 * p + 1] = s3[1];
      d.sdr[3 * p + 2] = s3[2];
    }
    ycc_bytes(s3, d.ycc + p, reinterpret_cast<int8_t*>(d.ycc + d.n) + p, reinterpret_cast<int8_t*>(d.ycc + 2 * d.n) + p);
  }
}

// Pass 2: the 8x8 DCT round trip of one tile = 8 pixel rows x 128 columns
// (16 blocks), everything in shared memory.  kDecode (the GPU decoder,
// decode.cu): start from the decoded zigzag coefficients instead, i.e. only
// _reconstruct (codec_core.py:478-489) -- the encoder's inverse half.
// out[o] = sum_t M[t][o] * in[t], t ascending, as idct_blocks (_kernels.py:404-422)
// sums it -- except that terms whose input is zero in every lane of the warp
// are skipped, and the sum starts at its first term rather than at 0.0.  A
// skipped term adds an exact zero, so every sum keeps its value (only the sign
// of a zero sum can differ, which no later rounding or clamp distinguishes).
// Chroma blocks at Q=85 are mostly zero above DC, so this removes most of
// their inverse-transform work.  All 32 lanes must call it.
__device__ __forceinline__ void idct_line(const double (&in)[8], double (&out)[8]) {
  unsigned m = 0;
#pragma unroll
  for (int tt = 0; tt < 8; tt++) m |= (in[tt] != 0.0 ? 1u : 0u) << tt;
  m = __reduce_or_sync(0xffffffffu, m);
#pragma unroll
  for (int o = 0; o < 8; o++) out[o] = 0.0;
  bool first = true;
#pragma unroll
  for (int tt = 0; tt < 8; tt++) {
    if (!(m & (1u << tt))) continue;
    if (first) {
#pragma unroll
      for (int o = 0; o < 8; o++) out[o] = kDctM[tt * 8 + o] * in[tt];
    } else {
#pragma unroll
      for (int o = 0; o < 8; o++) out[o] += kDctM[tt * 8 + o] * in[tt];
    }
    first = false;
  }
}

template <bool kDecode>
__global__ void __launch_bounds__(128, 8) k_base_layer(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int tiles_x = (d.nbx + kTileBlocks - 1) / kTileBlocks;
  const int tile = blockIdx.x;
  if (tile >= tiles_x * d.nby) return;
  const int by = tile / tiles_x;
  const int bx0 = (tile % tiles_x) * kTileBlocks;
  const int nblk = min(kTileBlocks, d.nbx - bx0);

  extern __shared__ double smem[];
  // [3][8][kRowStride], transformed in place: in every pass a thread reads its
  // whole line (a column or a row of one block) before writing it back, and
  // no two threads share a line within a pass
  double* bufA = smem;
  double* bufB = smem;
  const int t = threadIdx.x;

  // task t: block b = t / 8, line l = t % 8, for each of the 3 components
  const int b = t >> 3, l = t & 7;
  const bool live = b < nblk;
  const int col0 = b * 8;
  const long long bi = (long long)by * d.nbx + bx0 + b;

  if constexpr (kDecode) {  // dequantised coefficients, natural order (codec_core.py:481-483)
    if (live)
      for (int ci = 0; ci < 3; ci++) {
        const double* qt = d.qt + (ci == 0 ? 0 : 64);
        const int16_t* zz = d.zz + ((long long)ci * d.nblocks + bi) * 64;
#pragma unroll
        for (int v = 0; v < 8; v++)
          bufA[(ci * 8 + l) * kRowStride + col0 + v] = (double)zz[c_zigzag[l * 8 + v]] * qt[l * 8 + v];
      }
    __syncthreads();
  } else {
  // 1. the tile's YCC samples, edge-padded (np.pad mode="edge", codec_core.py:432-436)
  {
    const int rx = t;
    const int x = bx0 * 8 + rx, sx = min(x, d.w - 1);
    if (rx < nblk * 8) {
      const uint8_t* Yp = d.ycc;
      const int8_t* Cb = reinterpret_cast<const int8_t*>(d.ycc + d.n);
      const int8_t* Cr = reinterpret_cast<const int8_t*>(d.ycc + 2 * d.n);
#pragma unroll
      for (int ry = 0; ry < 8; ry++) {
        const long long pi = (long long)min(by * 8 + ry, d.h - 1) * d.w + sx;
        bufA[(0 * 8 + ry) * kRowStride + rx] = (double)__ldg(Yp + pi);
        bufA[(1 * 8 + ry) * kRowStride + rx] = (double)__ldg(Cb + pi);
        bufA[(2 * 8 + ry) * kRowStride + rx] = (double)__ldg(Cr + pi);
      }
    }
  }
  __syncthreads();

  // 2. forward pass 1 (dct_blocks first loop): tmp[u][x] = sum_t C[u][t] * blk[t][x], x = l
  if (live) {
#pragma unroll 1
    for (int ci = 0; ci < 3; ci++) {
      double in[8];
#pragma unroll
      for (int tt = 0; tt < 8; tt++) in[tt] = bufA[(ci * 8 + tt) * kRowStride + col0 + l];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        double s = kDctM[u * 8] * in[0];  // (0.0 + first term: same value up to the sign of a zero)
#pragma unroll
        for (int tt = 1; tt < 8; tt++) s += kDctM[u * 8 + tt] * in[tt];
        bufB[(ci * 8 + u) * kRowStride + col0 + l] = s;
      }
    }
  }
  __syncthreads();

  // 3. forward pass 2: out[u][v] = sum_t tmp[u][t] * C[v][t], u = l; quantise, zigzag, dequantise
  if (live) {
#pragma unroll 1
    for (int ci = 0; ci < 3; ci++) {
      const double* qt = d.qt + (ci == 0 ? 0 : 64);
      double in[8];
#pragma unroll
      for (int tt = 0; tt < 8; tt++) in[tt] = bufB[(ci * 8 + l) * kRowStride + col0 + tt];
      int16_t* zz = d.zz + ((long long)ci * d.nblocks + bi) * 64;
#pragma unroll
      for (int v = 0; v < 8; v++) {
        double s = in[0] * kDctM[v * 8];
#pragma unroll
        for (int tt = 1; tt < 8; tt++) s += in[tt] * kDctM[v * 8 + tt];
        const double qv = qt[l * 8 + v];
        const double qz = rha(s / qv);  // B200 fp64 division is cheaper than a certified reciprocal
        zz[c_zigzag[l * 8 + v]] = (int16_t)qz;
        bufA[(ci * 8 + l) * kRowStride + col0 + v] = qz * qv;  // dequantised coefficient
      }
    }
  }
  __syncthreads();

  }  // !kDecode

  // 4. inverse pass 1 (idct_blocks first loop): tmp[x][v] = sum_t C[t][x] * coef[t][v], v = l
#pragma unroll 1
  for (int ci = 0; ci < 3; ci++) {
    double in[8], out[8];
#pragma unroll
    for (int tt = 0; tt < 8; tt++) in[tt] = live ? bufA[(ci * 8 + tt) * kRowStride + col0 + l] : 0.0;
    idct_line(in, out);
    if (live)
#pragma unroll
      for (int x = 0; x < 8; x++) bufB[(ci * 8 + x) * kRowStride + col0 + l] = out[x];
  }
  __syncthreads();

  // 5. inverse pass 2: out[x][y] = sum_t tmp[x][t] * C[t][y], x = l
#pragma unroll 1
  for (int ci = 0; ci < 3; ci++) {
    double in[8], out[8];
#pragma unroll
    for (int tt = 0; tt < 8; tt++) in[tt] = live ? bufB[(ci * 8 + l) * kRowStride + col0 + tt] : 0.0;
    idct_line(in, out);
    if (live)
#pragma unroll
      for (int y = 0; y < 8; y++) bufA[(ci * 8 + l) * kRowStride + col0 + y] = out[y];
  }
  __syncthreads();

  // 6. _ycc_to_rgb on the cropped planes -> decoded S (3 planes)
  for (int p = t; p < 8 * kTileCols; p += blockDim.x) {
    int ry = p / kTileCols, rx = p % kTileCols;
    int y = by * 8 + ry, x = bx0 * 8 + rx;
    if (rx >= nblk * 8 || y >= d.h || x >= d.w) continue;
    double Y = bufA[(0 * 8 + ry) * kRowStride + rx];
    double cb = bufA[(1 * 8 + ry) * kRowStride + rx];
    double cr = bufA[(2 * 8 + ry) * kRowStride + rx];
    double v[3];
    v[0] = Y + 1.402 * cr;
    v[1] = Y - 0.344136 * cb - 0.714136 * cr;
    v[2] = Y + 1.772 * cb;
    long long pi = (long long)y * d.w + x;
#pragma unroll
    for (int c = 0; c < 3; c++) d.s_planes[c * d.n + pi] = (uint8_t)min(max(rha_int(v[c]), 0), 255);
  }
}

void upload_base_constants() {
  static const int zig[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                              12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                              35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                              58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
  // zz index k holds natural coefficient ZIGZAG[k]; the kernel scatters natural
  // position j to zz slot inv[j] where ZIGZAG[inv[j]] == j.
  int inv[64];
  for (int k = 0; k < 64; k++) inv[zig[k]] = k;
  cudaMemcpyToSymbol(c_zigzag, inv, sizeof(inv));
}

void launch_base_layer(const ImgDesc* d_descs, int nimg, int max_tiles, long long max_n, cudaStream_t st) {
  long long nq = (max_n + 3) / 4;
  int gx = (int)((nq + 255) / 256);
  if (gx > 148 * 8) gx = 148 * 8;
  if (gx < 1) gx = 1;
  k_sdr_ycc<<<dim3(gx, nimg), 256, 0, st>>>(d_descs);
  // ~0.3 % of the pixels, each an fp64 pow: about one CTA per 64 Ki pixels of the largest image
  const long long fx = std::min(1184LL, std::max(40LL, max_n >> 16));
  k_sdr_fix<<<dim3((unsigned)fx, nimg), 256, 0, st>>>(d_descs);
  size_t smem = sizeof(double) * 3 * 8 * kRowStride;
  cudaFuncSetAttribute(k_base_layer<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  // per device
  k_base_layer<false><<<dim3(max_tiles, nimg), 128, smem, st>>>(d_descs);
}

void launch_reconstruct(const ImgDesc* d_descs, int nimg, int max_tiles, cudaStream_t st) {
  size_t smem = sizeof(double) * 3 * 8 * kRowStride;
  cudaFuncSetAttribute(k_base_layer<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_base_layer<true><<<dim3(max_tiles, nimg), 128, smem, st>>>(d_descs);
}

}  // namespace hdll
