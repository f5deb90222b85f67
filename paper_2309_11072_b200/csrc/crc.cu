// crc.cu -- CRC-32 of the payload source data (codec_core.py:230-253).
//
// Each framed payload carries zlib.crc32 of the bytes the decoder must
// produce: the decoded interleaved RGB image for the base layer
// (codec_core.py:533) and the raw plane for each lossless payload (:313).
// Parallel form: every chunk (1 KiB of a plane, 256 pixels of the interleaved
// image) is CRC'd by one thread, slice-by-4 with each lane reading its own
// copy of the tables held in its own shared-memory bank (no bank conflicts:
// 128 KB, one 1024-thread CTA per SM), then chunks are merged with zlib's
// crc32_combine algebra: crc(A||B) = x^(8|B|) * crc(A) + crc(B) over GF(2) mod P.
#include <cstring>

#include "encoder.cuh"

namespace hdll {

__device__ uint32_t c_crc_tab[4][256];  // global, not __constant__: staged with divergent indices
__constant__ uint32_t c_x2n[32];  // x^(2^k) mod P, zlib x2n_table

__device__ __forceinline__ uint32_t x2nmodp(unsigned long long n, unsigned k) {
  uint32_t p = 1u << 31;  // x^0
  while (n) {
    if (n & 1) p = crc_multmodp(c_x2n[k & 31], p);
    n >>= 1;
    k++;
  }
  return p;
}

__device__ __forceinline__ uint32_t crc_combine(uint32_t a, uint32_t b, unsigned long long len_b) {
  return crc_multmodp(x2nmodp(len_b, 3), a) ^ b;
}

// job j of an image: 0 = decoded RGB interleaved (from S planes), 1 = E, 2..4 = residuals
// (over desc pixels [crc_p0, crc_p0 + crc_np): the whole image, or a row band's own rows)
__host__ __device__ __forceinline__ long long crc_job_len(const ImgDesc& d, int j) { return j == 0 ? 3 * d.crc_np : d.crc_np; }

__host__ __device__ __forceinline__ long long crc_chunk_bytes(int j) { return j == 0 ? kCrcChunkRgb : kCrcChunk; }

__host__ __device__ __forceinline__ long long crc_job_chunks(const ImgDesc& d, int j) {
  return (crc_job_len(d, j) + crc_chunk_bytes(j) - 1) / crc_chunk_bytes(j);
}

long long crc_assign_units(ImgDesc* ds, int n) {
  long long u = 0;
  for (int i = 0; i < n; i++) {
    ds[i].crc_u0 = u;
    for (int j = 0; j < 5; j++)
      if ((ds[i].crc_mask >> j) & 1) u += crc_job_chunks(ds[i], j);
  }
  return u;
}

constexpr int kCrcThreads = 1024;
constexpr size_t kCrcTabSmem = 4 * 256 * 32 * sizeof(uint32_t);  // [table][entry][lane]

// slice-by-4 on a lane's private tables (T = tabs + lane, entry stride 32 words)
__device__ __forceinline__ uint32_t crc_slice4(const uint32_t* T, uint32_t c, uint32_t w) {
  w ^= c;
  return T[(3 * 256 + (w & 0xFF)) * 32] ^ T[(2 * 256 + ((w >> 8) & 0xFF)) * 32] ^ T[(256 + ((w >> 16) & 0xFF)) * 32] ^
         T[(w >> 24) * 32];
}
__device__ __forceinline__ uint32_t crc_byte(const uint32_t* T, uint32_t c, uint32_t b) {
  return T[((c ^ b) & 0xFF) * 32] ^ (c >> 8);
}

// One work unit = one chunk of one job of one image, numbered through the
// batch (crc_u0); lane l of a warp takes unit 32 k + l, so whatever the image
// sizes every thread gets about the same number of bytes.
__global__ void __launch_bounds__(kCrcThreads, 1) k_crc_chunks(const ImgDesc* __restrict__ descs, int nimg, long long units) {
  extern __shared__ uint32_t tabs[];
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += blockDim.x) tabs[i] = (&c_crc_tab[0][0])[i >> 5];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t* T = tabs + lane;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long ub = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; ub < units; ub += nw * 32) {
    const long long u = ub + lane;
    if (u >= units) break;
    int lo = 0, hi = nimg;  // the image holding unit u: last crc_u0 <= u
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (descs[mid].crc_u0 <= u) lo = mid; else hi = mid;
    }
    const ImgDesc& d = descs[lo];
    long long chunk = u - d.crc_u0;
    int job = 0;
    for (; job < 5; job++) {
      if (!((d.crc_mask >> job) & 1)) continue;
      const long long nch = crc_job_chunks(d, job);
      if (chunk < nch) break;
      chunk -= nch;
    }
    if (job == 5) continue;  // (not reached: units are exact)
    const long long len = crc_job_len(d, job), csz = crc_chunk_bytes(job);
    const long long b0 = chunk * csz, nb = min(csz, len - b0);
    uint32_t c = 0xFFFFFFFFu;
    if (job == 0) {  // interleaved r g b of pixels [p0, p0 + nb / 3)
      const uint8_t* R = d.s_planes + d.crc_p0;
      const uint8_t* G = R + d.n;
      const uint8_t* B = G + d.n;
      const long long p0 = b0 / 3, np = nb / 3;
      long long p = p0;
      if (((reinterpret_cast<uintptr_t>(R + p0) | reinterpret_cast<uintptr_t>(G + p0) | reinterpret_cast<uintptr_t>(B + p0)) & 15) == 0) {
#pragma unroll 1
        for (; p + 16 <= p0 + np; p += 16) {
          const uint4 r4 = *reinterpret_cast<const uint4*>(R + p), g4 = *reinterpret_cast<const uint4*>(G + p),
                      b4 = *reinterpret_cast<const uint4*>(B + p);
          const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w}, gg[4] = {g4.x, g4.y, g4.z, g4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int h = 0; h < 4; h++) {
            const uint32_t r = rr[h], g = gg[h], b = bb[h];
            // little-endian words of the byte stream r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
            c = crc_slice4(T, c, __byte_perm(__byte_perm(r, g, 0x1040), b, 0x3410));
            c = crc_slice4(T, c, __byte_perm(__byte_perm(g, b, 0x2051), r, 0x3610));
            c = crc_slice4(T, c, __byte_perm(__byte_perm(b, r, 0x3072), g, 0x3710));
          }
        }
      }
      for (; p < p0 + np; p++) {
        c = crc_byte(T, c, R[p]);
        c = crc_byte(T, c, G[p]);
        c = crc_byte(T, c, B[p]);
      }
    } else {
      const uint8_t* q = (job == 1 ? d.e_plane : d.res_planes + (long long)(job - 2) * d.n) + d.crc_p0 + b0;
      long long k = 0;
      if ((reinterpret_cast<uintptr_t>(q) & 15) == 0) {
#pragma unroll 2
        for (; k + 16 <= nb; k += 16) {
          const uint4 v = *reinterpret_cast<const uint4*>(q + k);
          c = crc_slice4(T, c, v.x);
          c = crc_slice4(T, c, v.y);
          c = crc_slice4(T, c, v.z);
          c = crc_slice4(T, c, v.w);
        }
      }
      for (; k < nb; k++) c = crc_byte(T, c, q[k]);
    }
    d.crc_part[d.crc_part_off[job] + chunk] = c ^ 0xFFFFFFFFu;
  }
}

// One CTA (256 threads) per (image, job): each thread folds a run of `per`
// chunk CRCs (whole chunks through byte tables of x^(8 csz)), then a tree over
// the threads, whose regular right halves (per csz 2^s bytes) shift by a
// per-level constant.
constexpr int kCrcCombineThreads = 256;
__global__ void __launch_bounds__(kCrcCombineThreads) k_crc_combine(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int job = blockIdx.x;
  if (!((d.crc_mask >> job) & 1)) return;
  const long long len = crc_job_len(d, job);
  const long long csz = crc_chunk_bytes(job);
  const long long nch = (len + csz - 1) / csz;
  const uint32_t* part = d.crc_part + d.crc_part_off[job];
  constexpr int nt = kCrcCombineThreads;
  constexpr int kLevels = 8;  // log2(nt)
  const int t = threadIdx.x;
  __shared__ uint32_t scrc[nt];
  __shared__ unsigned long long slen[nt];
  __shared__ uint32_t xch[4][256];    // times x^(8 csz) (one whole chunk), as byte tables
  __shared__ uint32_t xlev[kLevels];  // times x^(8 per csz 2^s)
  __shared__ uint32_t xfull_s;
  const long long per = (nch + nt - 1) / nt;
  if (t < kLevels) xlev[t] = x2nmodp((unsigned long long)(per * csz) << t, 3);
  if (t == kLevels) xfull_s = x2nmodp((unsigned long long)csz, 3);
  __syncthreads();
  {
    const uint32_t xfull = xfull_s;
    for (int i = t; i < 1024; i += nt) xch[i >> 8][i & 255] = crc_multmodp(xfull, (uint32_t)(i & 255) << (8 * (i >> 8)));
  }
  __syncthreads();
  const long long c0 = (long long)t * per, c1 = min(nch, c0 + per);
  uint32_t acc = 0;
  unsigned long long alen = 0;
  if (c0 < c1) {
    acc = part[c0];
    alen = (unsigned long long)min(csz, len - c0 * csz);
    auto shift = [&](uint32_t a) {  // times x^(8 csz)
      return xch[0][a & 0xFF] ^ xch[1][(a >> 8) & 0xFF] ^ xch[2][(a >> 16) & 0xFF] ^ xch[3][a >> 24];
    };
    // whole chunks (all but the job's last), eight partial CRCs loaded ahead of their merges
    const long long cf = min(c1, nch - 1);
    long long k = c0 + 1;
    for (; k + 8 <= cf; k += 8) {
      uint32_t p8[8];
#pragma unroll
      for (int u = 0; u < 8; u++) p8[u] = part[k + u];
#pragma unroll
      for (int u = 0; u < 8; u++) acc = shift(acc) ^ p8[u];
      alen += 8ULL * (unsigned long long)csz;
    }
    for (; k < c1; k++) {
      unsigned long long l = (unsigned long long)min(csz, len - k * csz);
      if (l == (unsigned long long)csz) acc = shift(acc) ^ part[k];
      else acc = crc_multmodp(x2nmodp(l, 3), acc) ^ part[k];
      alen += l;
    }
  }
  scrc[t] = acc;
  slen[t] = alen;
  __syncthreads();
#pragma unroll 1
  for (int lv = 0; lv < kLevels; lv++) {
    const int sd = 1 << lv;
    if ((t & (2 * sd - 1)) == 0 && slen[t + sd] > 0) {
      const unsigned long long lr = slen[t + sd];
      if (!slen[t]) scrc[t] = scrc[t + sd];
      else if (lr == ((unsigned long long)(per * csz) << lv)) scrc[t] = crc_multmodp(xlev[lv], scrc[t]) ^ scrc[t + sd];
      else scrc[t] = crc_combine(scrc[t], scrc[t + sd], lr);
      slen[t] += lr;
    }
    __syncthreads();
  }
  if (t == 0) d.crc[job] = len ? scrc[0] : 0u;
}

void upload_crc_constants() {
  uint32_t tab[4][256];
  for (uint32_t i = 0; i < 256; i++) {
    uint32_t c = i;
    for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
    tab[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; i++)
    for (int t = 1; t < 4; t++) tab[t][i] = (tab[t - 1][i] >> 8) ^ tab[0][tab[t - 1][i] & 0xFF];
  uint32_t x2n[32];
  uint32_t p = 1u << 30;  // x^1
  x2n[0] = p;
  for (int n = 1; n < 32; n++) x2n[n] = p = crc_multmodp(p, p);
  cudaMemcpyToSymbol(c_crc_tab, tab, sizeof(tab));
  cudaMemcpyToSymbol(c_x2n, x2n, sizeof(x2n));
}

void launch_crc(const ImgDesc* d_descs, int nimg, long long units, cudaStream_t st) {
  if (units <= 0) return;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  cudaFuncSetAttribute(k_crc_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrcTabSmem);  // per device
  // one CTA per SM; no more warps than 32-unit groups
  long long gx = sms;
  const long long groups = (units + 31) / 32;
  if (gx * (kCrcThreads / 32) > groups) gx = (groups + kCrcThreads / 32 - 1) / (kCrcThreads / 32);
  k_crc_chunks<<<(unsigned)gx, kCrcThreads, kCrcTabSmem, st>>>(d_descs, nimg, units);
  k_crc_combine<<<dim3(5, nimg), kCrcCombineThreads, 0, st>>>(d_descs);
}

}  // namespace hdll
