// crc.cu -- CRC-32 of the payload source data (codec_core.py:230-253).
//
// Each framed payload carries zlib.crc32 of the bytes the decoder must
// produce: the decoded interleaved RGB image for the base layer
// (codec_core.py:533) and the raw plane for each lossless payload (:313).
// Parallel form: every 1 KiB chunk is CRC'd independently (slice-by-4 tables
// in shared memory), then chunks are merged with zlib's crc32_combine
// algebra: crc(A||B) = x^(8|B|) * crc(A) + crc(B) over GF(2) mod P.
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
// chunk bytes: whole pixels for the interleaved job (340 px), 1 KiB for planes
__host__ __device__ __forceinline__ long long crc_chunk_bytes(int j) { return j == 0 ? 1020 : kCrcChunk; }

__global__ void __launch_bounds__(256) k_crc_chunks(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int job = blockIdx.z;
  if (!((d.crc_mask >> job) & 1)) return;
  __shared__ uint32_t tab[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&tab[0][0])[i] = (&c_crc_tab[0][0])[i];
  __syncthreads();
  const long long len = crc_job_len(d, job);
  const long long csz = crc_chunk_bytes(job);
  const long long chunk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long b0 = chunk * csz;
  if (b0 >= len) return;
  const long long b1 = min(len, b0 + csz);
  uint32_t c = 0xFFFFFFFFu;
  if (job == 0) {
    // decoded RGB interleaved from the 3 S planes, 4 pixels (12 bytes) per step
    const uint8_t* R = d.s_planes + d.crc_p0;
    const uint8_t* G = d.s_planes + d.n + d.crc_p0;
    const uint8_t* B = d.s_planes + 2 * d.n + d.crc_p0;
    long long p = b0 / 3;
    const long long p1 = b1 / 3;  // chunks are whole pixels
    auto slice4 = [&](uint32_t w) {
      w ^= c;
      c = tab[3][w & 0xFF] ^ tab[2][(w >> 8) & 0xFF] ^ tab[1][(w >> 16) & 0xFF] ^ tab[0][w >> 24];
    };
    for (; p + 4 <= p1; p += 4) {
      uint32_t r4, g4, b4;
      memcpy(&r4, R + p, 4);
      memcpy(&g4, G + p, 4);
      memcpy(&b4, B + p, 4);
      // little-endian words of the byte stream r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
      slice4((r4 & 0xFF) | ((g4 & 0xFF) << 8) | ((b4 & 0xFF) << 16) | (((r4 >> 8) & 0xFF) << 24));
      slice4(((g4 >> 8) & 0xFF) | (((b4 >> 8) & 0xFF) << 8) | (((r4 >> 16) & 0xFF) << 16) |
             (((g4 >> 16) & 0xFF) << 24));
      slice4(((b4 >> 16) & 0xFF) | ((r4 >> 24) << 8) | ((g4 >> 24) << 16) | ((b4 >> 24) << 24));
    }
    for (; p < p1; p++) {
      c = tab[0][(c ^ R[p]) & 0xFF] ^ (c >> 8);
      c = tab[0][(c ^ G[p]) & 0xFF] ^ (c >> 8);
      c = tab[0][(c ^ B[p]) & 0xFF] ^ (c >> 8);
    }
  } else {
    const uint8_t* src = (job == 1 ? d.e_plane : d.res_planes + (long long)(job - 2) * d.n) + d.crc_p0;
    long long i = b0;
    // planes c > 0 start at c * n, which need not be word aligned
    for (; i < b1 && (reinterpret_cast<uintptr_t>(src + i) & 3); i++) c = tab[0][(c ^ src[i]) & 0xFF] ^ (c >> 8);
    for (; i + 4 <= b1; i += 4) {
      uint32_t w = *reinterpret_cast<const uint32_t*>(src + i) ^ c;
      c = tab[3][w & 0xFF] ^ tab[2][(w >> 8) & 0xFF] ^ tab[1][(w >> 16) & 0xFF] ^ tab[0][w >> 24];
    }
    for (; i < b1; i++) c = tab[0][(c ^ src[i]) & 0xFF] ^ (c >> 8);
  }
  d.crc_part[d.crc_part_off[job] + chunk] = c ^ 0xFFFFFFFFu;
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
}

void launch_crc(const ImgDesc* d_descs, int nimg, long long max_n, cudaStream_t st) {
  long long max_chunks = (3 * max_n + crc_chunk_bytes(0) - 1) / crc_chunk_bytes(0);
  k_crc_chunks<<<dim3((unsigned)((max_chunks + 255) / 256), nimg, 5), 256, 0, st>>>(d_descs);
  k_crc_combine<<<dim3(5, nimg), 1024, 0, st>>>(d_descs);
}

}  // namespace hdll
