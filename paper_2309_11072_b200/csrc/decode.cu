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

// MSB-first bit reader for one thread on a serial path.  `hi` always holds
// the next 64 bits of the stream, `lo` the nlo (32..63) bits after them; a
// consume of n <= 32 bits is one 64-bit funnel shift, and lo is topped up from
// a queue of two 32-bit words loaded ahead (branch-free), so no load sits on
// the dependency chain.  Bits past the body read as 0.  Reading past the end
// is detected lazily from the consumed bit count: the reference fails when a
// read starts or ends past the body (_kernels.py:82-111), and with zero
// padding the first such read ends past it too, so `pos > nbits` after the
// symbol is the same test; the callers check it at block / row boundaries and
// at the end, and every read until then stays inside the zero padding.
struct FastBits {
  const uint32_t* p;
  long long nw, wi;  // body words (the last one partial), next word to load
  uint32_t lastmask, q0, q1;
  unsigned long long hi, lo;
  int nlo;
  long long nbits;

  __device__ __forceinline__ uint32_t fetch() {  // branch-free: one clamped load, then selects
    const long long i = wi++;
    // (an empty body reads word 0 of its slot: every slot has 16 bytes of padding)
    const uint32_t w = __byte_perm(__ldg(p + (i < nw ? i : max(nw - 1, 0LL))), 0, 0x0123);
    return i < nw - 1 ? w : (i == nw - 1 ? (w & lastmask) : 0u);
  }
  __device__ __forceinline__ void init(const uint8_t* data, long long bytes) {
    p = reinterpret_cast<const uint32_t*>(data);  // 4-byte aligned (arena slot)
    nw = (bytes + 3) >> 2;
    const int tail = (int)(bytes & 3);
    lastmask = tail ? ~(0xFFFFFFFFu >> (8 * tail)) : 0xFFFFFFFFu;
    wi = 0;
    nbits = bytes * 8;
    const uint32_t a = fetch(), b = fetch(), c = fetch(), d = fetch();
    q0 = fetch();
    q1 = fetch();
    hi = ((unsigned long long)a << 32) | b;
    lo = ((unsigned long long)c << 32) | d;
    nlo = 64;
  }
  // bits consumed: the words moved into the window minus the window's bits
  __device__ __forceinline__ long long pos() const { return 32 * (wi - 2) - 64 - nlo; }
  __device__ __forceinline__ bool past_end() const { return pos() > nbits; }
  __device__ __forceinline__ uint32_t top() const { return (uint32_t)(hi >> 32); }
  // the 32 bits starting `off` (<= 32) bits into the window
  __device__ __forceinline__ uint32_t peek32(int off) const { return (uint32_t)(hi >> (32 - off)); }
  __device__ __forceinline__ void consume(int n) {  // 1 <= n <= 32
    hi = (hi << n) | (lo >> (64 - n));
    lo <<= n;
    nlo -= n;
    if (nlo < 32) {
      lo |= (unsigned long long)q0 << (32 - nlo);
      nlo += 32;
      q0 = q1;
      q1 = fetch();
    }
  }
  // _rice_get (_kernels.py:82-111): q ones, a zero, k bits; 24 ones: 8 raw bits
  __device__ __forceinline__ int rice(int k) {
    const uint32_t t = top();
    const int q = __clz(~t);
    const int len = q + 1 + k;
    if (q < kRiceEscapeQ && len <= 32) {
      const int u = (q << k) | (int)((t >> (32 - len)) & ((1u << k) - 1u));
      consume(len);
      return u;
    }
    return rice_slow(q, k);
  }
  __device__ __forceinline__ int rice_slow(int q, int k) {
    if (q >= kRiceEscapeQ) {
      const int u = (int)(top() & 0xFFu);
      consume(kRiceEscapeQ + 8);
      return u;
    }
    consume(q + 1);
    const int u = (q << k) | (int)(top() >> (32 - k));  // k >= 9 here
    consume(k);
    return u;
  }
  // s raw bits as the reference accumulates them (int64, wrapping)
  __device__ __forceinline__ long long raw(int s) {
    if (s <= 32) {
      const long long v = (long long)(top() >> (32 - s));
      consume(s);
      return v;
    }
    unsigned long long u = 0;
    long long r = s;
    while (r > 0) {
      const int k = (int)(r < 32 ? r : 32);
      u = (u << k) | (top() >> (32 - k));
      consume(k);
      r -= k;
      if (past_end()) break;  // the caller reports it
    }
    return (long long)u;
  }
};

// row buffer stride of the plane decoder: whole words and a spare byte for
// the one-sample-ahead load of the row above
__host__ __device__ __forceinline__ int dec_row_stride(int w) { return (w + 4) & ~3; }

// _select_k (_kernels.py:114-119): smallest k <= 15 with (N << k) >= A, closed
// form without branches (A < 2^31: u < 24 << 15 per symbol, and A halves every
// 32 symbols)
__device__ __forceinline__ int select_k_dec(int a, int n) {
  // bitlen(a-1) - bitlen(n), clamped to [0, 16] (16 and above all give 15, and
  // n << 16 < 2^22 for n <= 63, so the test stays in 32 bits)
  int k0 = min(max(__clz(n) - __clz(max(a - 1, 0)), 0), 16);
  k0 += (n << k0) < a ? 1 : 0;
  return min(k0, kRiceMaxK);
}

__device__ __forceinline__ int unzig32(int u) { return (u & 1) ? -((u + 1) >> 1) : (u >> 1); }
__device__ __forceinline__ long long unzig(long long u) { return (u & 1) == 0 ? (u >> 1) : -((u + 1) >> 1); }

// _update_state (_kernels.py:122-128) of one context held in registers, and
// the context's next Rice parameter
__device__ __forceinline__ void rice_update(int& A, int& N, int u) {
  A += u;
  N += 1;
  if (N >= kStateReset) {
    A >>= 1;
    N >>= 1;
  }
}

// decode_dct_component for the three components of one image (_kernels.py:327-378).
// Y uses contexts 0-2 and nothing after it does; Cb and Cr share 3-5
// (codec_core.py:439-450).  So one set of three context states in registers
// serves all three passes: reset before Y and before Cb, carried from Cb to Cr.
// An AC coefficient (zero run, size, raw bits) is decoded from the window in
// one straight pass when its codes fit 32 bits (nearly always): both Rice
// parameters are known before its bits are read.
__device__ __forceinline__ unsigned decode_dct_image(const ImgDesc& d) {
  FastBits br;
  br.init(d.pay[0], d.pay_bytes[0]);
  int Ad = 4, Nd = 1, Ar = 4, Nr = 1, As = 4, Ns = 1;  // DC size, zero run, AC size
  int kd = 2, kr = 2, ks = 2;                          // select_k(4, 1)
  uint32_t mr = 3u, ms = 3u;                           // (1 << k) - 1
#pragma unroll 1
  for (int ci = 0; ci < 3; ci++) {
    if (ci < 2) Ad = Ar = As = 4, Nd = Nr = Ns = 1, kd = kr = ks = 2, mr = ms = 3u;
    int16_t* zc = d.zz + (long long)ci * d.nblocks * 64;
    long long prev_dc = 0;
#pragma unroll 1
    for (long long b = 0; b < d.nblocks; b++) {
      int16_t* z = zc + b * 64;
      const int s = br.rice(kd);
      rice_update(Ad, Nd, s);
      kd = select_k_dec(Ad, Nd);
      const long long u = s > 0 ? br.raw(s) : 0;
      prev_dc += unzig(u);
      z[0] = (int16_t)prev_dc;
      int pos = 1;
#pragma unroll 1
      while (pos < 64) {
        // Fast path: zero run, size and raw bits of one coefficient read from
        // the top 64 bits without side effects, kept when all three fit the
        // top word and nothing is special (EOB, an escape, a corrupt value).
        const uint32_t t = (uint32_t)(br.hi >> 32), tl = (uint32_t)br.hi;
        const int q1 = __clz(~t);
        const int len1 = min(q1 + 1 + kr, 32);
        const int run = (q1 << kr) | (int)((t >> (32 - len1)) & mr);
        const uint32_t t2 = __funnelshift_lc(tl, t, len1);
        const int q2 = __clz(~t2);
        const int len2 = min(q2 + 1 + ks, 32);
        const int sz = (q2 << ks) | (int)((t2 >> (32 - len2)) & ms);
        const int L = len1 + len2;
        const int tot = L + sz;
        if (q1 < kRiceEscapeQ && q2 < kRiceEscapeQ && tot <= 32 && sz >= 1 && run < kEOB && pos + run <= 63) {
          const uint32_t v = (t << L) >> (32 - sz);  // L <= 31, 1 <= sz
          br.consume(tot);
          pos += run;
          z[pos] = (int16_t)unzig32((int)v);
          pos++;
          rice_update(Ar, Nr, run);
          kr = select_k_dec(Ar, Nr);
          mr = (1u << kr) - 1u;
          rice_update(As, Ns, sz);
          ks = select_k_dec(As, Ns);
          ms = (1u << ks) - 1u;
          continue;
        }
        // zero run (or EOB) one symbol at a time
        int rn;
        if (q1 < kRiceEscapeQ && q1 + 1 + kr <= 32) {
          rn = run;
          br.consume(len1);
        } else {
          rn = br.rice_slow(q1, kr);
        }
        rice_update(Ar, Nr, rn);
        kr = select_k_dec(Ar, Nr);
        mr = (1u << kr) - 1u;
        if (rn == kEOB) break;
        pos += rn;
        if (rn > 63 || pos > 63) return br.past_end() ? kDecTruncated : kDecCorrupt;
        const int sz1 = br.rice(ks);
        rice_update(As, Ns, sz1);
        ks = select_k_dec(As, Ns);
        ms = (1u << ks) - 1u;
        if (sz1 == 0 || sz1 > 62) return br.past_end() ? kDecTruncated : kDecCorrupt;
        z[pos] = (int16_t)unzig(br.raw(sz1));
        pos++;
      }
      if (br.past_end()) return kDecTruncated;
    }
  }
  return 0;
}

// decode_plane for one plane (kind 1 = E, 2..4 = residual R, G, B;
// _kernels.py:219-262).  The row above is kept in this thread's shared-memory
// buffers (the global copy was just written, so it would come back from L2 on
// the serial path).  The four regular contexts' states (A | N << 26: A stays
// below 2^26 even for u < 24 << 15 from a damaged stream, N <= 63) sit in shared memory, read as soon as the sample's
// context is known; their Rice parameters are kept in 4-bit fields of kp, so
// a sample's k is one shift after its context.
__device__ __forceinline__ unsigned decode_plane_dev(const ImgDesc& d, int kind, uint8_t* rows /* 2 * wpad */,
                                                     unsigned* sst /* 4 */) {
  uint8_t* P = kind == 1 ? d.e_plane : d.res_planes + (long long)(kind - 2) * d.n;
  FastBits br;
  br.init(d.pay[kind], d.pay_bytes[kind]);
  int Ar = 4, Nr = 1, krun = 2;  // the run context
  for (int i = 0; i < 4; i++) sst[i] = 4u | (1u << 26);
  uint32_t kp = 0x2222u;  // select_k(4, 1) = 2 for every context
  const int w = d.w;
  const int wpad = dec_row_stride(w);
  uint8_t* up = nullptr;
  uint8_t* cur = rows;
  for (int y = 0; y < d.h; y++) {
    uint8_t* grow = P + (long long)y * w;
    int x = 0;
    bool forced = false;
    int a = up ? up[0] : 128;  // a at x = 0 (_kernels.py:131-143)
    int bn = up ? up[0] : 0;   // b of the next sample, loaded a sample ahead
    int cp = bn;               // c: b of the previous sample (at x = 0, b itself)
#pragma unroll 1
    while (x < w) {
      const int b = up ? bn : a;
      const int c = up ? cp : a;
      if (up) bn = up[x + 1];  // (the row buffers have a spare byte)
      const bool runm = !forced && a == b && b == c;
      const int mx = max(a, b), mn = min(a, b);
      const int pred = c >= mx ? mn : (c <= mn ? mx : a + b - c);
      const int gg = abs(a - c) + abs(c - b);
      const int ctx = (gg > 0 ? 1 : 0) + (gg > 2 ? 1 : 0) + (gg > 8 ? 1 : 0);  // _activity_ctx
      const int k = (int)((kp >> (4 * ctx)) & 15u);
      const uint32_t t = br.top();
      const int q = __clz(~t);
      const int len = q + 1 + k;
      if (!runm) {
        unsigned st = sst[ctx];
        int u;
        if (q < kRiceEscapeQ && len <= 32) {
          u = (q << k) | (int)((t >> (32 - len)) & ((1u << k) - 1u));
          br.consume(len);
        } else {
          u = br.rice_slow(q, k);
        }
        const int v = (pred + unzig32(u)) & 255;
        cur[x] = (uint8_t)v;
        grow[x] = (uint8_t)v;
        {  // _update_state: A += u, N += 1; at N = 64 both halve
          const unsigned n = st >> 26;
          const unsigned A = (st & 0x3FFFFFFu) + (unsigned)u;
          st = n == kStateReset - 1 ? (A >> 1) | ((unsigned)(kStateReset / 2) << 26) : A | ((n + 1) << 26);
          sst[ctx] = st;
          const int sh = 4 * ctx;
          kp = (kp & ~(15u << sh)) | ((uint32_t)select_k_dec((int)(st & 0x3FFFFFFu), (int)(st >> 26)) << sh);
        }
        cp = b;
        a = v;
        x++;
        forced = false;
        continue;
      }
      int run = 0;
      for (;;) {
        const int chunk = br.rice(krun);
        rice_update(Ar, Nr, chunk);
        krun = select_k_dec(Ar, Nr);
        run += chunk;
        if (chunk < 255) break;
        if (run > w) break;  // corrupt either way; bounded
      }
      if (x + run > w) return br.past_end() ? kDecTruncated : kDecCorrupt;
      for (int i = 0; i < run; i++) {
        cur[x + i] = (uint8_t)a;
        grow[x + i] = (uint8_t)a;
      }
      x += run;
      if (x < w) forced = true;
      if (up) {  // the look-ahead already moved past x (a run may be empty)
        cp = up[x > 0 ? x - 1 : 0];
        bn = up[x];
      }
    }
    if (br.past_end()) return kDecTruncated;
    up = cur;
    cur = cur == rows ? rows + wpad : rows;
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
  else if (with_planes) {
    __shared__ unsigned dec_state[4][4];
    st = decode_plane_dev(d, t, dec_rows + (long long)(t - 1) * 2 * dec_row_stride(max_w), dec_state[t - 1]);
  }
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
  const size_t smem = planes ? (size_t)8 * dec_row_stride(max_w) : 0;
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
