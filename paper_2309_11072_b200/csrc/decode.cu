// decode.cu -- GPU decoder: decode_hdr / decode_sdr (container.py:233-280).
//
// The two adaptive-Rice decoders are sequential by format (each symbol's Rice
// parameter depends on every earlier symbol of its stream), so each stream is
// decoded by one thread -- one per image for the base layer (decode_dct_component,
// _kernels.py:327-378, the three components in turn with shared contexts), one
// per (image, plane) for the four lossless planes (decode_plane,
// _kernels.py:219-262) -- and the batch supplies the parallelism.  Everything
// after the coders is data parallel and reuses the encoder's kernels:
// _reconstruct (base.cu k_base_layer<true>), the prefilter, the M* estimate
// (here M = (M* + r) & 255 straight into RGBE quads) and the CRC-32 checks of
// the frames.  Device status bits per image: 1 << (16 + k) when stream k ends
// early or is inconsistent (the reference's CorruptPayloadError), 1 << 21 when
// an exponent has no regression entry (StreamError); CRC mismatches are
// compared on the host.
#include "encoder.cuh"

namespace hdll {

enum : uint32_t { kDecTruncated = 1u, kDecCorrupt = 2u, kDecBadShift = 16, kDecNoEntry = 1u << 21 };

// MSB-first bit reader with a 64-bit window; bits past the body read as 0 and
// `avail` tells how many real bits remain (the reference fails on reading past
// the end: _kernels.py:82-111).
struct BitReader {
  const uint32_t* p;       // the body, 4-byte aligned (staged so by the host)
  long long nbytes, next;  // next byte to load (a multiple of 4 while words remain)
  unsigned long long win;  // left-aligned
  int have;                // bits in win that came from the body

  __device__ __forceinline__ void init(const uint8_t* data, long long bytes) {
    p = reinterpret_cast<const uint32_t*>(data);
    nbytes = bytes;
    next = 0;
    win = 0;
    have = 0;
    refill();
  }
  // whole big-endian words while they fit; the last partial word is masked to
  // the body (bytes past it read as 0 and do not count in `have`)
  __device__ __forceinline__ void refill() {
    while (have <= 32 && next < nbytes) {
      const uint32_t w = __byte_perm(__ldg(p + (next >> 2)), 0, 0x0123);
      const long long left = nbytes - next;
      const int nb = left >= 4 ? 4 : (int)left;
      const uint32_t wm = nb == 4 ? w : (w & ~(0xFFFFFFFFu >> (8 * nb)));
      win |= (unsigned long long)wm << (32 - have);
      have += 8 * nb;
      next += nb;
    }
  }
  __device__ __forceinline__ unsigned long long take(int k) {  // k in [1, 32], have >= k
    const unsigned long long v = win >> (64 - k);
    win <<= k;
    have -= k;
    return v;
  }
  // _rice_get (_kernels.py:82-111); -1 when the body ends first
  __device__ __forceinline__ long long rice(int k) {
    refill();
    const int ones = __clzll(~win);  // zero bits past `have` stop the count
    if (ones >= kRiceEscapeQ) {
      if (have < kRiceEscapeQ + 8) return -1;
      take(kRiceEscapeQ);
      return (long long)take(8);
    }
    if (ones >= have) return -1;  // ran out before the terminating zero
    if (have < ones + 1 + k) return -1;
    take(ones + 1);
    long long u = (long long)ones << k;
    if (k) u |= (long long)take(k);
    return u;
  }
  // s raw bits as the reference accumulates them (int64, wrapping)
  __device__ __forceinline__ long long raw(long long s, bool* ok) {
    long long u = 0;
    while (s > 0) {
      refill();
      const int k = (int)(s < 32 ? s : 32);
      if (have < k) {
        *ok = false;
        return 0;
      }
      u = (long long)(((unsigned long long)u << k) | take(k));
      s -= k;
    }
    return u;
  }
};

// _select_k (_kernels.py:114-119): smallest k <= 15 with (N << k) >= A, closed form
// (A < 2^31: u < 24 << 15 per symbol, and A halves every 32 symbols)
__device__ __forceinline__ int select_k_dec(int a, int n) {
  if (a <= n) return 0;
  const int k0 = __clz(n) - __clz(a - 1);  // bitlen(a-1) - bitlen(n) >= 0
  const int k = (((long long)n << k0) >= a) ? k0 : k0 + 1;
  return k < kRiceMaxK ? k : kRiceMaxK;
}

// Adaptive-Rice state of NC contexts in registers (no local-memory arrays on
// the serial path); _update_state (_kernels.py:122-128)
template <int NC>
struct RiceState {
  int A[NC], N[NC];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int i = 0; i < NC; i++) A[i] = 4, N[i] = 1;
  }
  __device__ __forceinline__ int k(int c) const {
    int a = A[0], n = N[0];
#pragma unroll
    for (int i = 1; i < NC; i++)
      if (c == i) a = A[i], n = N[i];
    return select_k_dec(a, n);
  }
  __device__ __forceinline__ void update(int c, long long u) {
#pragma unroll
    for (int i = 0; i < NC; i++)
      if (c == i) {
        A[i] += (int)u;
        N[i] += 1;
        if (N[i] >= kStateReset) {
          A[i] >>= 1;
          N[i] >>= 1;
        }
      }
  }
};

__device__ __forceinline__ long long unzig(long long u) { return (u & 1) == 0 ? (u >> 1) : -((u + 1) >> 1); }

// decode_dct_component for the three components of one image
__device__ unsigned decode_dct_image(const ImgDesc& d) {
  BitReader br;
  br.init(d.pay[0], d.pay_bytes[0]);
  RiceState<6> rs;
  rs.reset();
#pragma unroll  // the contexts become compile-time register indices
  for (int ci = 0; ci < 3; ci++) {
    const int base = ci == 0 ? 0 : 3;
    int16_t* zc = d.zz + (long long)ci * d.nblocks * 64;
    long long prev_dc = 0;
    for (long long b = 0; b < d.nblocks; b++) {
      int16_t* z = zc + b * 64;
      long long s = br.rice(rs.k(base));
      if (s < 0) return kDecTruncated;
      rs.update(base, s);
      bool ok = true;
      const long long u = s > 0 ? br.raw(s, &ok) : 0;
      if (!ok) return kDecTruncated;
      prev_dc += unzig(u);
      z[0] = (int16_t)prev_dc;
      int pos = 1;
      while (pos < 64) {
        const long long run = br.rice(rs.k(base + 1));
        if (run < 0) return kDecTruncated;
        rs.update(base + 1, run);
        if (run == kEOB) break;
        pos += (int)run;
        if (run > 63 || pos > 63) return kDecCorrupt;
        s = br.rice(rs.k(base + 2));
        if (s < 0) return kDecTruncated;
        rs.update(base + 2, s);
        if (s == 0 || s > 62) return kDecCorrupt;
        const long long v = br.raw(s, &ok);
        if (!ok) return kDecTruncated;
        z[pos] = (int16_t)unzig(v);
        pos++;
      }
    }
  }
  return 0;
}

// decode_plane for one plane (kind 1 = E, 2..4 = residual R, G, B); the row
// above is kept in this thread's shared-memory buffers (the global copy was
// just written, so it would come back from L2 on the serial path)
__device__ unsigned decode_plane_dev(const ImgDesc& d, int kind, uint8_t* rows /* 2 * w */) {
  uint8_t* P = kind == 1 ? d.e_plane : d.res_planes + (long long)(kind - 2) * d.n;
  BitReader br;
  br.init(d.pay[kind], d.pay_bytes[kind]);
  RiceState<5> rs;
  rs.reset();
  const int w = d.w;
  uint8_t* up = nullptr;
  uint8_t* cur = rows;
  for (int y = 0; y < d.h; y++) {
    uint8_t* grow = P + (long long)y * w;
    int x = 0;
    bool forced = false;
    int left = up ? up[0] : 128;  // a at x = 0 (_kernels.py:131-143)
    while (x < w) {
      const int a = left;
      const int b = up ? up[x] : a;
      const int c = (up && x > 0) ? up[x - 1] : b;
      if (!forced && a == b && b == c) {
        long long run = 0;
        for (;;) {
          const long long chunk = br.rice(rs.k(kRunCtx));
          if (chunk < 0) return kDecTruncated;
          rs.update(kRunCtx, chunk);
          run += chunk;
          if (chunk < 255) break;
        }
        if (x + run > w) return kDecCorrupt;
        for (long long i = 0; i < run; i++) {
          cur[x + i] = (uint8_t)a;
          grow[x + i] = (uint8_t)a;
        }
        x += (int)run;
        if (x < w) forced = true;
        continue;
      }
      const int mx = max(a, b), mn = min(a, b);
      const int pred = c >= mx ? mn : (c <= mn ? mx : a + b - c);
      const int gg = abs(a - c) + abs(c - b);
      const int ctx = gg == 0 ? 0 : (gg <= 2 ? 1 : (gg <= 8 ? 2 : 3));
      const long long u = br.rice(rs.k(ctx));
      if (u < 0) return kDecTruncated;
      const int v = (int)((pred + unzig(u)) & 255);
      cur[x] = (uint8_t)v;
      grow[x] = (uint8_t)v;
      left = v;
      rs.update(ctx, u);
      x++;
      forced = false;
    }
    up = cur;
    cur = cur == rows ? rows + w : rows;
  }
  return 0;
}

// one thread per stream, each in its own warp (lanes of one warp would take
// turns on their divergent paths): warp 0 of image i's block decodes the base
// layer, warps 1..4 its planes (each with 2 rows of dynamic shared memory)
__global__ void __launch_bounds__(160) k_decode_coders(const ImgDesc* __restrict__ descs, int with_planes, int max_w) {
  extern __shared__ uint8_t dec_rows[];
  const ImgDesc& d = descs[blockIdx.x];
  if (threadIdx.x & 31) return;
  const int t = threadIdx.x >> 5;
  if (d.crc_mask == 0x2 && t != 1) return;  // plane-only job: body 1 alone
  unsigned st = 0;
  if (t == 0) st = decode_dct_image(d);
  else if (with_planes) st = decode_plane_dev(d, t, dec_rows + (long long)(t - 1) * 2 * max_w);
  if (st) atomicOr(d.status, 1u << (kDecBadShift + t));
}

// M = (M* + r) & 255 with M* from the estimate (container.py:245-268), written
// as RGBE quads with the decoded E; or, for an SDR decode, S interleaved.
__global__ void __launch_bounds__(256) k_decode_output(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  __shared__ float sa[3 * 256], sb[3 * 256];
  const bool sdr_only = d.crc_mask == 1;
  if (d.slrme && !sdr_only)
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) {
      sa[i] = d.a32[i];
      sb[i] = d.b32[i];
    }
  __syncthreads();
  const bool real = d.sigma_milli != 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < d.n; p += (long long)gridDim.x * blockDim.x) {
    if (d.crc_mask == 0x2) {  // plane-only job: the decoded plane itself
      d.out_rgbe[p] = d.e_plane[p];
      continue;
    }
    if (sdr_only) {
#pragma unroll
      for (int c = 0; c < 3; c++) d.out_rgbe[3 * p + c] = d.s_planes[(long long)c * d.n + p];
      continue;
    }
    const unsigned e = d.e_plane[p];
    uint32_t q = e << 24;
#pragma unroll
    for (int c = 0; c < 3; c++) {
      unsigned ms;
      if (d.slrme) {
        const double s = real ? d.sstar[(long long)c * d.n + p] : (double)d.s_planes[(long long)c * d.n + p];
        const float a = sa[c * 256 + e];
        if (isnan(a)) atomicOr(d.status, kDecNoEntry);  // absent entry (estimator.py:82-92 KeyError)
        const double est = (double)a * s + (double)sb[c * 256 + e];
        ms = (unsigned)min(max(rha_int(est), 0), 255);
      } else {
        ms = d.s_planes[(long long)c * d.n + p];
      }
      q |= ((ms + d.res_planes[(long long)c * d.n + p]) & 255u) << (8 * c);
    }
    reinterpret_cast<uint32_t*>(d.out_rgbe)[p] = q;
  }
}

void launch_decode_coders(const ImgDesc* d_descs, int nimg, bool planes, int max_w, cudaStream_t st) {
  const size_t smem = planes ? (size_t)8 * max_w : 0;
  cudaFuncSetAttribute(k_decode_coders, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_decode_coders<<<nimg, planes ? 160 : 32, smem, st>>>(d_descs, planes ? 1 : 0, max_w);
}

void launch_decode_output(const ImgDesc* d_descs, int nimg, long long max_n, cudaStream_t st) {
  long long gx = (max_n + 255) / 256;
  const long long cap = (148 * 8 + nimg - 1) / nimg;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  k_decode_output<<<dim3((unsigned)gx, nimg), 256, 0, st>>>(d_descs);
}

}  // namespace hdll
