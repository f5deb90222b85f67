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
      unsigned long long bits = k == 0 ? at.dct_bits[img] : at.plane_bits[img * 4 + k - 1];
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
  }
  __syncthreads();
  const long long total = min(L.total, d.out_cap);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
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
      if (r < 17) v = frame[k][r];
      else v = (k == 0 ? at.dct_out[img] : at.plane_out[img * 4 + k - 1])[r - 17];
    }
    d.out[i] = v;
  }
}

void launch_assemble(const ImgDesc* d_descs, int nimg, const AsmTab& at, long long max_out, cudaStream_t st) {
  long long blocks = (max_out + 256 * 16 - 1) / (256 * 16);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_assemble<<<dim3((unsigned)blocks, nimg), 256, 0, st>>>(d_descs, at);
}

}  // namespace hdll
