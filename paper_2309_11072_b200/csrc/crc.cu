// crc.cu -- CRC-32 of the payload source data (codec_core.py:230-253).
//
// Each framed payload carries zlib.crc32 of the bytes the decoder must
// produce: the decoded interleaved RGB image for the base layer
// (codec_core.py:533) and the raw plane for each lossless payload (:313).
// Parallel form: every 1 KiB chunk is CRC'd independently (slice-by-4 tables
// in shared memory), then chunks are merged with zlib's crc32_combine
// algebra: crc(A||B) = x^(8|B|) * crc(A) + crc(B) over GF(2) mod P.
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
__device__ __forceinline__ long long crc_job_len(const ImgDesc& d, int j) { return j == 0 ? 3 * d.n : d.n; }

__global__ void __launch_bounds__(256) k_crc_chunks(const ImgDesc* __restrict__ descs) {
  const ImgDesc& d = descs[blockIdx.y];
  const int job = blockIdx.z;
  if (!((d.crc_mask >> job) & 1)) return;
  __shared__ uint32_t tab[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&tab[0][0])[i] = (&c_crc_tab[0][0])[i];
  __syncthreads();
  const long long len = crc_job_len(d, job);
  const long long chunk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long b0 = chunk * kCrcChunk;
  if (b0 >= len) return;
  const long long b1 = min(len, b0 + kCrcChunk);
  uint32_t c = 0xFFFFFFFFu;
  if (job == 0) {
    const uint8_t* S = d.s_planes;
    long long p = b0 / 3;
    int ch = (int)(b0 % 3);
    for (long long i = b0; i < b1; i++) {
      uint8_t byte = S[(long long)ch * d.n + p];
      c = tab[0][(c ^ byte) & 0xFF] ^ (c >> 8);
      if (++ch == 3) {
        ch = 0;
        p++;
      }
    }
  } else {
    const uint8_t* src = job == 1 ? d.e_plane : d.res_planes + (long long)(job - 2) * d.n;
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
  const long long nch = (len + kCrcChunk - 1) / kCrcChunk;
  const uint32_t* part = d.crc_part + d.crc_part_off[job];
  const int nt = blockDim.x, t = threadIdx.x;
  __shared__ uint32_t scrc[1024];
  __shared__ unsigned long long slen[1024];
  const long long per = (nch + nt - 1) / nt;
  const long long c0 = (long long)t * per, c1 = min(nch, c0 + per);
  uint32_t acc = 0;
  unsigned long long alen = 0;
  if (c0 < c1) {
    const uint32_t xfull = x2nmodp((unsigned long long)kCrcChunk, 3);
    acc = part[c0];
    alen = (unsigned long long)min((long long)kCrcChunk, len - c0 * kCrcChunk);
    for (long long k = c0 + 1; k < c1; k++) {
      unsigned long long l = (unsigned long long)min((long long)kCrcChunk, len - k * kCrcChunk);
      uint32_t xp = (l == (unsigned long long)kCrcChunk) ? xfull : x2nmodp(l, 3);
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
  long long max_chunks = (3 * max_n + kCrcChunk - 1) / kCrcChunk;
  k_crc_chunks<<<dim3((unsigned)((max_chunks + 255) / 256), nimg, 5), 256, 0, st>>>(d_descs);
  k_crc_combine<<<dim3(5, nimg), 1024, 0, st>>>(d_descs);
}

}  // namespace hdll
