// crc.cu -- CRC-32 of the payload source data (codec_core.py:230-253).
//
// Each framed payload carries zlib.crc32 of the bytes the decoder must
// produce: the decoded interleaved RGB image for the base layer
// (codec_core.py:533) and the raw plane for each lossless payload (:313).
// Parallel form: every chunk (1 KiB of a plane, 256 pixels of the interleaved
// image) is CRC'd by one warp (slice-by-4 tables in shared memory, one piece
// per lane, pieces merged in-warp), then chunks are merged with zlib's
// crc32_combine algebra: crc(A||B) = x^(8|B|) * crc(A) + crc(B) over GF(2) mod P.
#include <cstring>

#include "encoder.cuh"

namespace hdll {

__constant__ uint32_t c_crc_tab[4][256];
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
__device__ __forceinline__ long long crc_job_len(const ImgDesc& d, int j) { return j == 0 ? 3 * d.crc_np : d.crc_np; }

// A chunk is the bytes of one warp: 32 lanes x kCrcLaneBytes[j] contiguous
// bytes (8 whole pixels = 24 bytes for the interleaved job, 32 bytes of a
// plane).  Lanes CRC their pieces, then the warp merges them in log2(32)
// steps with crc(A||B) = x^(8|B|) crc(A) + crc(B); multiplying by the fixed
// x^(8 P 2^k) is a GF(2)-linear map applied through four 256-entry tables.
constexpr int kCrcLaneBytesRgb = kCrcChunkRgb / 32, kCrcLaneBytesPlane = kCrcChunk / 32;
__host__ __device__ __forceinline__ long long crc_lane_bytes(int j) { return j == 0 ? kCrcLaneBytesRgb : kCrcLaneBytesPlane; }
__host__ __device__ __forceinline__ long long crc_chunk_bytes(int j) { return 32 * crc_lane_bytes(j); }

__device__ uint32_t c_shift_tab[2][5][4][256];  // [rgb / plane][k][byte][value]: times x^(8 P 2^k)

__device__ __forceinline__ uint32_t crc_bytes(const uint32_t (*tab)[256], uint32_t c, const uint8_t* p, int n) {
  for (int i = 0; i < n; i++) c = tab[0][(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c;
}

__global__ void __launch_bounds__(256) k_crc_chunks(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int job = blockIdx.z;
  if (!((d.crc_mask >> job) & 1)) return;
  __shared__ uint32_t tab[4][256];
  __shared__ uint32_t sht[5][4][256];
  const int kind = job == 0 ? 0 : 1;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&tab[0][0])[i] = (&c_crc_tab[0][0])[i];
  for (int i = threadIdx.x; i < 5 * 1024; i += blockDim.x) (&sht[0][0][0])[i] = (&c_shift_tab[kind][0][0][0])[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long len = crc_job_len(d, job);
  const long long csz = crc_chunk_bytes(job), lb = crc_lane_bytes(job);
  const long long nch = (len + csz - 1) / csz;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  auto slice4 = [&](uint32_t c, uint32_t w) {
    w ^= c;
    return tab[3][w & 0xFF] ^ tab[2][(w >> 8) & 0xFF] ^ tab[1][(w >> 16) & 0xFF] ^ tab[0][w >> 24];
  };
  const uint8_t* R = d.s_planes + d.crc_p0;
  const uint8_t* G = d.s_planes + d.n + d.crc_p0;
  const uint8_t* B = d.s_planes + 2 * d.n + d.crc_p0;
  const uint8_t* src = job == 0 ? nullptr : (job == 1 ? d.e_plane : d.res_planes + (long long)(job - 2) * d.n) + d.crc_p0;
  for (long long chunk = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); chunk < nch; chunk += wstride) {
    const long long b0 = chunk * csz;
    if (b0 + csz > len) {  // the job's last, partial chunk: one lane, byte by byte
      if (lane == 0) {
        uint32_t c = 0xFFFFFFFFu;
        if (job == 0) {
          for (long long p = b0 / 3; p < len / 3; p++) {
            const uint8_t px[3] = {R[p], G[p], B[p]};
            c = crc_bytes(tab, c, px, 3);
          }
        } else {
          c = crc_bytes(tab, c, src + b0, (int)(len - b0));
        }
        d.crc_part[d.crc_part_off[job] + chunk] = c ^ 0xFFFFFFFFu;
      }
      continue;
    }
    uint32_t c = 0xFFFFFFFFu;
    const long long o = b0 + lane * lb;
    if (job == 0) {  // 8 pixels: 3 plane words each, interleaved r g b
      const long long p = o / 3;
      uint32_t r[2], g[2], bb[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        memcpy(&r[h], R + p + 4 * h, 4);
        memcpy(&g[h], G + p + 4 * h, 4);
        memcpy(&bb[h], B + p + 4 * h, 4);
      }
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t r4 = r[h], g4 = g[h], b4 = bb[h];
        // little-endian words of the byte stream r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
        c = slice4(c, (r4 & 0xFF) | ((g4 & 0xFF) << 8) | ((b4 & 0xFF) << 16) | (((r4 >> 8) & 0xFF) << 24));
        c = slice4(c, ((g4 >> 8) & 0xFF) | (((b4 >> 8) & 0xFF) << 8) | (((r4 >> 16) & 0xFF) << 16) |
                          (((g4 >> 16) & 0xFF) << 24));
        c = slice4(c, ((b4 >> 16) & 0xFF) | ((r4 >> 24) << 8) | ((g4 >> 24) << 16) | ((b4 >> 24) << 24));
      }
    } else {
      uint32_t w[8];
      const uint8_t* q = src + o;
      if ((reinterpret_cast<uintptr_t>(q) & 15) == 0) {
        const uint4 v0 = *reinterpret_cast<const uint4*>(q), v1 = *reinterpret_cast<const uint4*>(q + 16);
        w[0] = v0.x, w[1] = v0.y, w[2] = v0.z, w[3] = v0.w, w[4] = v1.x, w[5] = v1.y, w[6] = v1.z, w[7] = v1.w;
      } else {
#pragma unroll
        for (int k = 0; k < 8; k++) memcpy(&w[k], q + 4 * k, 4);
      }
#pragma unroll
      for (int k = 0; k < 8; k++) c = slice4(c, w[k]);
    }
    c ^= 0xFFFFFFFFu;
    // merge: at step k, lanes 2^(k+1) i hold the CRC of 2^k pieces, their right
    // neighbours the next 2^k pieces
#pragma unroll
    for (int k = 0; k < 5; k++) {
      const uint32_t right = __shfl_down_sync(0xffffffffu, c, 1 << k);
      if ((lane & ((2 << k) - 1)) == 0)
        c = sht[k][0][c & 0xFF] ^ sht[k][1][(c >> 8) & 0xFF] ^ sht[k][2][(c >> 16) & 0xFF] ^ sht[k][3][c >> 24] ^ right;
    }
    if (lane == 0) d.crc_part[d.crc_part_off[job] + chunk] = c;
  }
}

// one CTA (1024 threads) per (image, job): sequential runs then a tree
__global__ void __launch_bounds__(1024) k_crc_combine(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int job = blockIdx.x;
  if (!((d.crc_mask >> job) & 1)) return;
  const long long len = crc_job_len(d, job);
  const long long csz = crc_chunk_bytes(job);
  const long long nch = (len + csz - 1) / csz;
  const uint32_t* part = d.crc_part + d.crc_part_off[job];
  const int nt = blockDim.x, t = threadIdx.x;
  __shared__ uint32_t scrc[1024];
  __shared__ unsigned long long slen[1024];
  const long long per = (nch + nt - 1) / nt;
  const long long c0 = (long long)t * per, c1 = min(nch, c0 + per);
  uint32_t acc = 0;
  unsigned long long alen = 0;
  if (c0 < c1) {
    const uint32_t xfull = x2nmodp((unsigned long long)csz, 3);
    acc = part[c0];
    alen = (unsigned long long)min(csz, len - c0 * csz);
    for (long long k = c0 + 1; k < c1; k++) {
      unsigned long long l = (unsigned long long)min(csz, len - k * csz);
      uint32_t xp = (l == (unsigned long long)csz) ? xfull : x2nmodp(l, 3);
      acc = crc_multmodp(xp, acc) ^ part[k];
      alen += l;
    }
  }
  scrc[t] = acc;
  slen[t] = alen;
  __syncthreads();
  for (int s = 1; s < nt; s <<= 1) {
    if ((t % (2 * s)) == 0 && slen[t + s] > 0) {
      scrc[t] = slen[t] ? crc_combine(scrc[t], scrc[t + s], slen[t + s]) : scrc[t + s];
      slen[t] += slen[t + s];
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
  // shift tables: x^(8 len) mod P for len = P 2^k, as byte-indexed linear maps
  static uint32_t sh[2][5][4][256];
  for (int kind = 0; kind < 2; kind++)
    for (int k = 0; k < 5; k++) {
      unsigned long long n = (unsigned long long)(kind == 0 ? kCrcLaneBytesRgb : kCrcLaneBytesPlane) << k;
      uint32_t x = 1u << 31;  // x^0; x^(8 n) by square-and-multiply over x2n
      unsigned kk = 3;
      while (n) {
        if (n & 1) x = crc_multmodp(x2n[kk & 31], x);
        n >>= 1;
        kk++;
      }
      for (int b = 0; b < 4; b++)
        for (uint32_t v = 0; v < 256; v++) sh[kind][k][b][v] = crc_multmodp(x, v << (8 * b));
    }
  cudaMemcpyToSymbol(c_shift_tab, sh, sizeof(sh));
}

void launch_crc(const ImgDesc* d_descs, int nimg, long long max_n, cudaStream_t st) {
  long long max_chunks = (3 * max_n + crc_chunk_bytes(0) - 1) / crc_chunk_bytes(0);
  // 8 warps per CTA looping over chunks: few CTAs per (image, job), since each
  // first stages 24 KB of tables in shared memory
  long long gx = (max_chunks + 63) / 64;
  const long long cap = (148 * 8 + 5 * nimg - 1) / (5 * nimg);
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  k_crc_chunks<<<dim3((unsigned)gx, nimg, 5), 256, 0, st>>>(d_descs);
  k_crc_combine<<<dim3(5, nimg), 1024, 0, st>>>(d_descs);
}

}  // namespace hdll
