// assemble.cu -- serialize() on the device (container.py:306-340).
//
//   fixed header + TMO record       host-built bytes (hdr_pre)
//   u16 count + count x <BBffI      regression table, sorted by (channel, exponent)
//   u32 len + header text block     host-built bytes (hdr_post)
//   5 framed payloads               <IBI (5 + len(body), coder id, crc32) + body,
//                                   body = <II (w, h) + MSB-first bits (codec_core.py:230-231,
//                                   :263-265, :451)
// Every CTA recomputes the (tiny) layout and copies its slice of output bytes.
#include "encoder.cuh"

namespace hdll {

struct Layout {
  long long pre, tab, post, pay[5], body_len[5], total;
  int npresent;
};

__device__ __forceinline__ void put_le32(uint8_t* p, uint32_t v) {
  p[0] = v & 0xFF;
  p[1] = (v >> 8) & 0xFF;
  p[2] = (v >> 16) & 0xFF;
  p[3] = v >> 24;
}

__device__ __forceinline__ uint32_t be_word(const uint8_t* p, long long k) {
  return __byte_perm(reinterpret_cast<const uint32_t*>(p)[k], 0, 0x0123);
}

// 32 bits of an MSB-first stream of `nbits` bits from bit `b` (>= 0) on; bits
// past the end read as 0
__device__ __forceinline__ uint32_t bits_at(const uint8_t* p, long long nbits, long long b) {
  if (b >= nbits) return 0u;
  const long long k = b >> 5;
  const int sh = (int)(b & 31);
  uint32_t v = be_word(p, k) << sh;
  if (sh && (k + 1) * 32 < nbits) v |= be_word(p, k + 1) >> (32 - sh);
  const long long valid = nbits - b;
  if (valid < 32) v &= ~0u << (32 - valid);
  return v;
}

// Little-endian word k (stream bytes 4k .. 4k+3) of the base-layer body when
// it is two chains: Y's bits, then Cb, Cr's bits straight after them.
__device__ __forceinline__ uint32_t split_word(const uint8_t* y, long long ybits, const uint8_t* c, long long cbits,
                                               long long k) {
  const long long o = 32 * k;
  uint32_t v;
  if (o + 32 <= ybits) v = be_word(y, k);
  else if (o >= ybits) v = bits_at(c, cbits, o - ybits);
  else v = bits_at(y, ybits, o) | (bits_at(c, cbits, 0) >> (int)(ybits - o));
  return __byte_perm(v, 0, 0x0123);
}

__global__ void __launch_bounds__(256) k_assemble(const ImgDesc* __restrict__ descs, AsmTab at) {
  const ImgDesc& d = descs[blockIdx.y];
  __shared__ Layout L;
  __shared__ uint8_t present[256];
  __shared__ int prefix[257];
  __shared__ uint8_t frame[5][17];
  const int img = blockIdx.y;
  if (threadIdx.x < 256) present[threadIdx.x] = (d.slrme && d.bin_count[threadIdx.x] > 0) ? 1 : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < 256; e++) {
      prefix[e] = run;
      run += present[e];
    }
    prefix[256] = run;
    L.npresent = run;
    long long o = 0;
    L.pre = o;
    o += d.hdr_pre_len;
    L.tab = o;
    o += 2 + 14LL * 3 * run;
    L.post = o;
    o += d.hdr_post_len;
    for (int k = 0; k < 5; k++) {
      const unsigned long long bits =
          k == 0 ? at.dct_bits[img * at.dct_stride] + (at.dct_split ? at.dct_bits[img * at.dct_stride + 1] : 0ULL)
                 : at.plane_bits[img * 4 + k - 1];
      L.body_len[k] = 8 + (long long)((bits + 7) / 8);
      L.pay[k] = o;
      o += 9 + L.body_len[k];
      // frame: <IBI> then <II> w, h ; payload order: base, E, R, G, B; crc jobs 0..4 match
      put_le32(frame[k], (uint32_t)(5 + L.body_len[k]));
      frame[k][4] = 1;
      put_le32(frame[k] + 5, d.crc[k]);
      put_le32(frame[k] + 9, (uint32_t)d.w);
      put_le32(frame[k] + 13, (uint32_t)d.h);
    }
    L.total = o;
    if (blockIdx.x == 0) *d.out_len = (unsigned long long)o;
    if (o > d.out_cap) atomicOr(d.status, kErrCapacity);
    // every earlier stage of this batch has finished (stream order); fold the
    // image's status into the context's accumulated word
    if (blockIdx.x == 0 && at.err_acc) {
      const unsigned s = *(volatile unsigned*)d.status;
      if (s) atomicOr(at.err_acc, s);
    }
  }
  __syncthreads();
  const long long total = min(L.total, d.out_cap);
  // payload bit streams: the bulk, copied 16 bytes at a time (funnel shifts
  // re-align the 4-byte aligned source to the byte offset in the stream)
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < 5; k++) {
    const uint8_t* src = k == 0 ? at.dct_out[img * at.dct_stride] : at.plane_out[img * 4 + k - 1];
    const long long dst0 = L.pay[k] + 17, len = L.body_len[k] - 8;
    if (k == 0 && at.dct_split) {  // Y chain + Cb, Cr chain, bit-contiguous
      const uint8_t* cs = at.dct_out[img * at.dct_stride + 1];
      const long long yb = (long long)at.dct_bits[img * at.dct_stride];
      const long long cb = (long long)at.dct_bits[img * at.dct_stride + 1];
      const long long head = min(len, (16 - ((long long)(reinterpret_cast<uintptr_t>(d.out) + dst0) & 15)) & 15);
      for (long long i = tid; i < head; i += nthreads)
        if (dst0 + i < total) d.out[dst0 + i] = (uint8_t)(split_word(src, yb, cs, cb, i >> 2) >> (8 * (i & 3)));
      const long long nvec = (len - head) / 16;
      for (long long v = tid; v < nvec; v += nthreads) {
        const long long so = head + v * 16;
        const long long k0 = so >> 2;
        const int sh = (int)(so & 3);
        uint32_t w[5];
#pragma unroll
        for (int q = 0; q < 5; q++) w[q] = (q < 4 || sh) ? split_word(src, yb, cs, cb, k0 + q) : 0u;
        uint4 o;
        o.x = __funnelshift_r(w[0], w[1], 8 * sh);
        o.y = __funnelshift_r(w[1], w[2], 8 * sh);
        o.z = __funnelshift_r(w[2], w[3], 8 * sh);
        o.w = __funnelshift_r(w[3], w[4], 8 * sh);
        if (dst0 + so + 16 <= total) *reinterpret_cast<uint4*>(d.out + dst0 + so) = o;
      }
      for (long long i = head + nvec * 16 + tid; i < len; i += nthreads)
        if (dst0 + i < total) d.out[dst0 + i] = (uint8_t)(split_word(src, yb, cs, cb, i >> 2) >> (8 * (i & 3)));
      continue;
    }
    // head bytes up to a 16-byte aligned destination, then aligned 16-byte chunks
    const long long head = min(len, (16 - ((long long)(reinterpret_cast<uintptr_t>(d.out) + dst0) & 15)) & 15);
    for (long long i = tid; i < head; i += nthreads)
      if (dst0 + i < total) d.out[dst0 + i] = src[i];
    const long long nvec = (len - head) / 16;
    for (long long v = tid; v < nvec; v += nthreads) {
      const long long so = head + v * 16;  // source byte offset
      const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src + (so & ~3LL));
      const int sh = (int)(so & 3);
      uint32_t w[5];
#pragma unroll
      for (int q = 0; q < 5; q++) w[q] = (q < 4 || sh) ? s4[q] : 0u;
      uint4 o;
      // little-endian byte stream: byte b of the output = source byte so + b
      o.x = __funnelshift_r(w[0], w[1], 8 * sh);
      o.y = __funnelshift_r(w[1], w[2], 8 * sh);
      o.z = __funnelshift_r(w[2], w[3], 8 * sh);
      o.w = __funnelshift_r(w[3], w[4], 8 * sh);
      if (dst0 + so + 16 <= total) *reinterpret_cast<uint4*>(d.out + dst0 + so) = o;
    }
    for (long long i = head + nvec * 16 + tid; i < len; i += nthreads)
      if (dst0 + i < total) d.out[dst0 + i] = src[i];
  }
  // everything else (headers, table, frames): byte by byte
  for (long long i = tid; i < total; i += nthreads) {
    uint8_t v;
    if (i < L.tab) {
      v = d.hdr_pre[i];
    } else if (i < L.post) {
      long long r = i - L.tab;
      if (r < 2) {
        int cnt = 3 * L.npresent;
        v = r == 0 ? (cnt & 0xFF) : (cnt >> 8);
      } else {
        long long k = (r - 2) / 14;
        int f = (int)((r - 2) % 14);
        int ch = (int)(k / L.npresent);
        int j = (int)(k % L.npresent);
        int lo = 0, hi = 256;  // exponent with prefix[e] == j and present
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (prefix[mid] <= j) lo = mid; else hi = mid;
        }
        int e = lo;
        uint32_t word;
        if (f == 0) {
          v = (uint8_t)ch;
        } else if (f == 1) {
          v = (uint8_t)e;
        } else {
          if (f < 6) word = __float_as_uint(d.a32[ch * 256 + e]);
          else if (f < 10) word = __float_as_uint(d.b32[ch * 256 + e]);
          else word = d.bin_count[e];
          int byte = (f - 2) & 3;
          v = (word >> (8 * byte)) & 0xFF;
        }
      }
    } else if (i < L.pay[0]) {
      v = d.hdr_post[i - L.post];
    } else {
      int k = 4;
      while (i < L.pay[k]) k--;
      long long r = i - L.pay[k];
      if (r >= 17) {  // bit-stream bytes were written above
        long long skip = L.pay[k] + 9 + L.body_len[k] - i;  // jump to the next frame
        i += skip - 1 - ((skip - 1) % nthreads);
        continue;
      }
      v = frame[k][r];
    }
    d.out[i] = v;
  }
}

// ---------------------------------------------------------------------------
// Bit concatenation (tile-sharded images): piece p's nbits[p] MSB-first bits
// are OR-ed into dst at bit dst_bit[p].  Words shared with a neighbouring
// piece (a piece's first and last) use atomicOr; dst starts zeroed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bitcat(uint8_t* dst, const uint8_t* const* src,
                                                const unsigned long long* dst_bit, const unsigned long long* nbits) {
  const int piece = blockIdx.y;
  const long long L = (long long)nbits[piece];
  if (L == 0) return;
  const long long o = (long long)dst_bit[piece];
  const uint8_t* sp = src[piece];
  const long long w0 = o >> 5, w1 = (o + L - 1) >> 5, last_src = (L - 1) >> 5;
  uint32_t* out = reinterpret_cast<uint32_t*>(dst);
  for (long long w = w0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; w <= w1;
       w += (long long)gridDim.x * blockDim.x) {
    const long long off = 32 * w - o;  // source bit at the word's first bit
    uint32_t v;
    if (off < 0) {
      v = be_word(sp, 0) >> (int)(-off);
    } else {
      const long long k = off >> 5;
      const int sh = (int)(off & 31);
      v = be_word(sp, k) << sh;
      if (sh && k + 1 <= last_src) v |= be_word(sp, k + 1) >> (32 - sh);
    }
    const long long valid = L - off;  // source bits left from the word's first bit
    if (valid < 32) v &= ~0u << (32 - valid);
    const uint32_t le = __byte_perm(v, 0, 0x0123);
    if (w == w0 || w == w1) atomicOr(out + w, le);
    else out[w] = le;
  }
}

void launch_bitcat(uint8_t* dst, const uint8_t* const* src, const unsigned long long* dst_bit,
                   const unsigned long long* nbits, int npieces, unsigned long long max_bits, cudaStream_t st) {
  if (npieces <= 0) return;
  long long words = (long long)(max_bits / 32) + 2;
  long long bx = (words + 255) / 256;
  if (bx > 148 * 4) bx = 148 * 4;
  if (bx < 1) bx = 1;
  k_bitcat<<<dim3((unsigned)bx, npieces), 256, 0, st>>>(dst, src, dst_bit, nbits);
}

void launch_assemble(const ImgDesc* d_descs, int nimg, const AsmTab& at, long long max_out, cudaStream_t st) {
  // ~64 KiB per CTA, and about 8 CTAs per SM over the whole batch: every CTA
  // recomputes the (small) layout first
  long long blocks = (max_out + 65535) / 65536;
  const long long cap = (148 * 8 + nimg - 1) / nimg;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_assemble<<<dim3((unsigned)blocks, nimg), 256, 0, st>>>(d_descs, at);
}

}  // namespace hdll
