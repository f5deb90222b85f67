/*
 * hdll_oracle.c -- CPU restatement of the reference encoder's loops.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product path (paper_2309_11072_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It is never
 * linked into, or called by, the product.
 *
 * It restates, in plain C with the exact floating-point operation order of the
 * reference (numpy / scipy / numba / OpenBLAS as used by /root/reference/pkg),
 * every loop of hdll.container.encode except the tone-map transcendental pass,
 * which oracle/hdll_oracle.py restates with numpy itself (same ufuncs as the
 * reference).  Citations are to /root/reference/pkg/src/hdll/<file>:<line>.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: no FMA contraction; the
 * only fused multiply-adds are the explicit fma() calls that model OpenBLAS).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RICE_MAX_K 15    /* _kernels.py:13 */
#define RICE_ESCAPE_Q 24 /* _kernels.py:14 */
#define STATE_RESET 64   /* _kernels.py:15 */
#define PLANE_CTX 5      /* _kernels.py:16 */
#define RUN_CTX 4        /* _kernels.py:17 */
#define DCT_CTX 6        /* _kernels.py:18 */
#define EOB 64           /* _kernels.py:19 */

/* ------------------------------------------------------------------------- */
/* CRC-32 (zlib.crc32, codec_core.py:252-253): reflected poly 0xEDB88320.     */
/* ------------------------------------------------------------------------- */
static uint32_t crc_table[8][256];
static pthread_once_t crc_once = PTHREAD_ONCE_INIT;

static void crc_init(void) {
  for (uint32_t i = 0; i < 256; i++) {
    uint32_t c = i;
    for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
    crc_table[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; i++)
    for (int t = 1; t < 8; t++)
      crc_table[t][i] = (crc_table[t - 1][i] >> 8) ^ crc_table[0][crc_table[t - 1][i] & 0xFF];
}

uint32_t ho_crc32(const uint8_t *p, size_t n) {
  pthread_once(&crc_once, crc_init);
  uint32_t c = 0xFFFFFFFFu;
  while (n >= 8) { /* slice-by-8 */
    uint32_t lo = c ^ ((uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24);
    uint32_t hi = (uint32_t)p[4] | (uint32_t)p[5] << 8 | (uint32_t)p[6] << 16 | (uint32_t)p[7] << 24;
    c = crc_table[7][lo & 0xFF] ^ crc_table[6][(lo >> 8) & 0xFF] ^ crc_table[5][(lo >> 16) & 0xFF] ^
        crc_table[4][lo >> 24] ^ crc_table[3][hi & 0xFF] ^ crc_table[2][(hi >> 8) & 0xFF] ^
        crc_table[1][(hi >> 16) & 0xFF] ^ crc_table[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = (c >> 8) ^ crc_table[0][(c ^ *p++) & 0xFF];
  return c ^ 0xFFFFFFFFu;
}

/* ------------------------------------------------------------------------- */
/* MSB-first bit writer (_kernels.py:46-57; codec_core.py:95-124).            */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint8_t *buf; /* zero-initialised, capacity checked by the caller */
  uint64_t pos; /* bit position */
} bw_t;

static inline void bw_put(bw_t *w, uint64_t v, int n) {
  for (int i = n - 1; i >= 0; i--) {
    if ((v >> i) & 1) w->buf[w->pos >> 3] |= (uint8_t)(1u << (7 - (w->pos & 7)));
    w->pos++;
  }
}

static inline void bw_ones(bw_t *w, int n) {
  for (int i = 0; i < n; i++) {
    w->buf[w->pos >> 3] |= (uint8_t)(1u << (7 - (w->pos & 7)));
    w->pos++;
  }
}

/* _rice_put, _kernels.py:65-79 */
static inline void rice_put(bw_t *w, int64_t u, int k) {
  int64_t q = u >> k;
  if (q < RICE_ESCAPE_Q) {
    bw_ones(w, (int)q);
    w->pos++; /* the terminating zero */
    if (k > 0) bw_put(w, (uint64_t)(u & ((1 << k) - 1)), k);
  } else {
    bw_ones(w, RICE_ESCAPE_Q);
    bw_put(w, (uint64_t)u, 8);
  }
}

typedef struct {
  const uint8_t *data;
  uint64_t nbits;
  uint64_t pos;
} br_t;

static inline int br_bit(br_t *r) { return (r->data[r->pos >> 3] >> (7 - (r->pos & 7))) & 1; }

/* _rice_get, _kernels.py:82-111: returns -1 on truncation */
static int64_t rice_get(br_t *r, int k) {
  int64_t q = 0;
  for (;;) {
    if (r->pos >= r->nbits) return -1;
    int bit = br_bit(r);
    r->pos++;
    if (bit == 0) break;
    q++;
    if (q == RICE_ESCAPE_Q) {
      if (r->pos + 8 > r->nbits) return -1;
      int64_t u = 0;
      for (int i = 0; i < 8; i++) {
        u = (u << 1) | br_bit(r);
        r->pos++;
      }
      return u;
    }
  }
  int64_t u = q << k;
  if (k > 0) {
    if (r->pos + (uint64_t)k > r->nbits) return -1;
    int64_t rr = 0;
    for (int i = 0; i < k; i++) {
      rr = (rr << 1) | br_bit(r);
      r->pos++;
    }
    u |= rr;
  }
  return u;
}

/* _select_k / _update_state, _kernels.py:114-128 */
static inline int select_k(int64_t a, int64_t n) {
  int k = 0;
  while ((n << k) < a && k < RICE_MAX_K) k++;
  return k;
}

static inline void update_state(int64_t *A, int64_t *N, int ctx, int64_t u) {
  A[ctx] += u;
  N[ctx] += 1;
  if (N[ctx] >= STATE_RESET) {
    A[ctx] >>= 1;
    N[ctx] >>= 1;
  }
}

/* ------------------------------------------------------------------------- */
/* Lossless plane coder id 1 (_kernels.py:131-262)                            */
/* ------------------------------------------------------------------------- */
static inline void neighbors(const uint8_t *p, int w, int y, int x, int64_t *a, int64_t *b, int64_t *c) {
  /* _kernels.py:131-143 */
  if (x > 0)
    *a = p[(size_t)y * w + x - 1];
  else if (y > 0)
    *a = p[(size_t)(y - 1) * w + x];
  else
    *a = 128;
  *b = (y > 0) ? p[(size_t)(y - 1) * w + x] : *a;
  *c = (x > 0 && y > 0) ? p[(size_t)(y - 1) * w + x - 1] : *b;
}

static inline int64_t med(int64_t a, int64_t b, int64_t c) { /* _kernels.py:146-154 */
  int64_t mx = a > b ? a : b, mn = a < b ? a : b;
  if (c >= mx) return mn;
  if (c <= mn) return mx;
  return a + b - c;
}

static inline int activity_ctx(int64_t a, int64_t b, int64_t c) { /* _kernels.py:157-166 */
  int64_t g = llabs(a - c) + llabs(c - b);
  if (g == 0) return 0;
  if (g <= 2) return 1;
  if (g <= 8) return 2;
  return 3;
}

/* encode_plane, _kernels.py:169-216.  out must hold h*w*8+128 bytes, zeroed
 * here.  Returns the bit count; the byte length is (bits+7)/8. */
uint64_t ho_encode_plane(const uint8_t *plane, int h, int w, uint8_t *out) {
  size_t cap = (size_t)h * w * 8 + 128;
  memset(out, 0, cap);
  bw_t bw = {out, 0};
  int64_t A[PLANE_CTX], N[PLANE_CTX];
  for (int i = 0; i < PLANE_CTX; i++) A[i] = 4, N[i] = 1;
  for (int y = 0; y < h; y++) {
    const uint8_t *row = plane + (size_t)y * w;
    int x = 0, forced = 0;
    while (x < w) {
      int64_t a, b, c;
      neighbors(plane, w, y, x, &a, &b, &c);
      if (!forced && a == b && b == c) {
        int run = 0;
        while (x + run < w && (int64_t)row[x + run] == a) run++;
        int rem = run;
        for (;;) {
          int chunk = rem >= 255 ? 255 : rem;
          rice_put(&bw, chunk, select_k(A[RUN_CTX], N[RUN_CTX]));
          update_state(A, N, RUN_CTX, chunk);
          rem -= chunk;
          if (chunk < 255) break;
        }
        x += run;
        if (x < w) forced = 1;
        continue;
      }
      int64_t pred = med(a, b, c);
      int ctx = activity_ctx(a, b, c);
      int64_t r = ((int64_t)row[x] - pred) & 255;
      if (r > 127) r -= 256;
      int64_t u = r >= 0 ? 2 * r : -2 * r - 1;
      rice_put(&bw, u, select_k(A[ctx], N[ctx]));
      update_state(A, N, ctx, u);
      x++;
      forced = 0;
    }
  }
  return bw.pos;
}

/* decode_plane, _kernels.py:219-262.  Returns status 0 ok, 1 truncated, 2 corrupt. */
int ho_decode_plane(const uint8_t *data, size_t nbytes, int h, int w, uint8_t *plane) {
  br_t br = {data, (uint64_t)nbytes * 8, 0};
  memset(plane, 0, (size_t)h * w);
  int64_t A[PLANE_CTX], N[PLANE_CTX];
  for (int i = 0; i < PLANE_CTX; i++) A[i] = 4, N[i] = 1;
  for (int y = 0; y < h; y++) {
    int x = 0, forced = 0;
    while (x < w) {
      int64_t a, b, c;
      neighbors(plane, w, y, x, &a, &b, &c);
      if (!forced && a == b && b == c) {
        int64_t run = 0;
        for (;;) {
          int64_t chunk = rice_get(&br, select_k(A[RUN_CTX], N[RUN_CTX]));
          if (chunk < 0) return 1;
          update_state(A, N, RUN_CTX, chunk);
          run += chunk;
          if (chunk < 255) break;
        }
        if (x + run > w) return 2;
        for (int64_t i = 0; i < run; i++) plane[(size_t)y * w + x + i] = (uint8_t)a;
        x += (int)run;
        if (x < w) forced = 1;
        continue;
      }
      int64_t pred = med(a, b, c);
      int ctx = activity_ctx(a, b, c);
      int64_t u = rice_get(&br, select_k(A[ctx], N[ctx]));
      if (u < 0) return 1;
      int64_t r = (u & 1) == 0 ? (u >> 1) : -((u + 1) >> 1);
      plane[(size_t)y * w + x] = (uint8_t)((pred + r) & 255);
      update_state(A, N, ctx, u);
      x++;
      forced = 0;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Lossy coder id 1: 8x8 block DCT (codec_core.py:336-489, _kernels.py:21-43, */
/* 265-422).                                                                 */
/* ------------------------------------------------------------------------- */
static const double DCT_M[8][8] = { /* _kernels.py:23-43 */
    {0.35355339059327373, 0.35355339059327373, 0.35355339059327373, 0.35355339059327373,
     0.35355339059327373, 0.35355339059327373, 0.35355339059327373, 0.35355339059327373},
    {0.4903926402016152, 0.4157348061512726, 0.27778511650980114, 0.09754516100806417,
     -0.0975451610080641, -0.277785116509801, -0.4157348061512727, -0.4903926402016152},
    {0.46193976625564337, 0.19134171618254492, -0.19134171618254486, -0.46193976625564337,
     -0.4619397662556434, -0.19134171618254517, 0.191341716182545, 0.46193976625564326},
    {0.4157348061512726, -0.0975451610080641, -0.4903926402016152, -0.2777851165098011,
     0.2777851165098009, 0.4903926402016152, 0.09754516100806439, -0.41573480615127256},
    {0.3535533905932738, -0.35355339059327373, -0.35355339059327384, 0.3535533905932737,
     0.35355339059327384, -0.35355339059327334, -0.35355339059327356, 0.3535533905932733},
    {0.27778511650980114, -0.4903926402016152, 0.09754516100806415, 0.41573480615127273,
     -0.41573480615127256, -0.09754516100806401, 0.4903926402016153, -0.27778511650980076},
    {0.19134171618254492, -0.4619397662556434, 0.46193976625564326, -0.19134171618254495,
     -0.19134171618254528, 0.46193976625564337, -0.4619397662556432, 0.19134171618254478},
    {0.09754516100806417, -0.2777851165098011, 0.41573480615127273, -0.4903926402016153,
     0.4903926402016152, -0.4157348061512725, 0.27778511650980076, -0.09754516100806429},
};

static const int ZIGZAG[64] = { /* codec_core.py:364-372 */
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
    41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
    30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

static const double LUMA_QT[64] = { /* codec_core.py:337-349 */
    16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
    14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
    18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
static const double CHROMA_QT[64] = { /* codec_core.py:350-362 */
    17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99, 24, 26, 56, 99, 99, 99,
    99, 99, 47, 66, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99};

/* round_half_away, _util.py:8-11: trunc(x + copysign(0.5, x)) */
static inline double rha(double x) { return trunc(x + copysign(0.5, x)); }

/* quantization_tables, codec_core.py:375-388 */
void ho_quant_tables(int quality, double *luma, double *chroma) {
  double scale = quality < 50 ? 5000.0 / quality : 200.0 - 2.0 * quality;
  for (int i = 0; i < 64; i++) {
    double t = rha(LUMA_QT[i] * scale / 100.0);
    luma[i] = t < 1 ? 1 : (t > 255 ? 255 : t);
    t = rha(CHROMA_QT[i] * scale / 100.0);
    chroma[i] = t < 1 ? 1 : (t > 255 ? 255 : t);
  }
}

/* dct_blocks, _kernels.py:381-400 (one block, fixed order, no FMA) */
static void dct8x8(const double *blk, double *out) {
  double tmp[64];
  for (int u = 0; u < 8; u++)
    for (int x = 0; x < 8; x++) {
      double s = 0.0;
      for (int t = 0; t < 8; t++) s += DCT_M[u][t] * blk[t * 8 + x];
      tmp[u * 8 + x] = s;
    }
  for (int u = 0; u < 8; u++)
    for (int v = 0; v < 8; v++) {
      double s = 0.0;
      for (int t = 0; t < 8; t++) s += tmp[u * 8 + t] * DCT_M[v][t];
      out[u * 8 + v] = s;
    }
}

/* idct_blocks, _kernels.py:403-422 */
static void idct8x8(const double *coef, double *out) {
  double tmp[64];
  for (int x = 0; x < 8; x++)
    for (int v = 0; v < 8; v++) {
      double s = 0.0;
      for (int t = 0; t < 8; t++) s += DCT_M[t][x] * coef[t * 8 + v];
      tmp[x * 8 + v] = s;
    }
  for (int x = 0; x < 8; x++)
    for (int y = 0; y < 8; y++) {
      double s = 0.0;
      for (int t = 0; t < 8; t++) s += tmp[x * 8 + t] * DCT_M[t][y];
      out[x * 8 + y] = s;
    }
}

static inline int bit_length(int64_t u) { /* _kernels.py:270-277 */
  int s = 0;
  while (u > 0) u >>= 1, s++;
  return s;
}
static inline int64_t interleave(int64_t v) { return v >= 0 ? 2 * v : -2 * v - 1; }

/* encode_dct_component, _kernels.py:280-324 */
static void encode_dct_component(bw_t *bw, const int64_t *zz, size_t nblocks, int cls, int64_t *A, int64_t *N) {
  int base = cls * 3;
  int64_t prev_dc = 0;
  for (size_t i = 0; i < nblocks; i++) {
    const int64_t *z = zz + i * 64;
    int64_t d = z[0] - prev_dc;
    prev_dc = z[0];
    int64_t u = interleave(d);
    int s = bit_length(u);
    rice_put(bw, s, select_k(A[base], N[base]));
    update_state(A, N, base, s);
    if (s > 0) bw_put(bw, (uint64_t)u, s);
    int pos = 1;
    while (pos < 64) {
      int nz = -1;
      for (int j = pos; j < 64; j++)
        if (z[j] != 0) {
          nz = j;
          break;
        }
      if (nz < 0) {
        rice_put(bw, EOB, select_k(A[base + 1], N[base + 1]));
        update_state(A, N, base + 1, EOB);
        break;
      }
      int run = nz - pos;
      rice_put(bw, run, select_k(A[base + 1], N[base + 1]));
      update_state(A, N, base + 1, run);
      u = interleave(z[nz]);
      s = bit_length(u);
      rice_put(bw, s, select_k(A[base + 2], N[base + 2]));
      update_state(A, N, base + 2, s);
      bw_put(bw, (uint64_t)u, s);
      pos = nz + 1;
    }
  }
}

/* decode_dct_component, _kernels.py:327-378 */
static int decode_dct_component(br_t *br, int64_t *zz, size_t nblocks, int cls, int64_t *A, int64_t *N) {
  int base = cls * 3;
  int64_t prev_dc = 0;
  memset(zz, 0, nblocks * 64 * sizeof(int64_t));
  for (size_t i = 0; i < nblocks; i++) {
    int64_t *z = zz + i * 64;
    int64_t s = rice_get(br, select_k(A[base], N[base]));
    if (s < 0) return 1;
    update_state(A, N, base, s);
    int64_t u = 0;
    if (s > 0) {
      if (br->pos + (uint64_t)s > br->nbits) return 1;
      for (int64_t t = 0; t < s; t++) {
        u = (u << 1) | br_bit(br);
        br->pos++;
      }
    }
    int64_t d = (u & 1) == 0 ? (u >> 1) : -((u + 1) >> 1);
    prev_dc += d;
    z[0] = prev_dc;
    int pos = 1;
    while (pos < 64) {
      int64_t run = rice_get(br, select_k(A[base + 1], N[base + 1]));
      if (run < 0) return 1;
      update_state(A, N, base + 1, run);
      if (run == EOB) break;
      pos += (int)run;
      if (pos > 63) return 2;
      s = rice_get(br, select_k(A[base + 2], N[base + 2]));
      if (s < 0) return 1;
      update_state(A, N, base + 2, s);
      if (s == 0 || s > 62) return 2;
      if (br->pos + (uint64_t)s > br->nbits) return 1;
      u = 0;
      for (int64_t t = 0; t < s; t++) {
        u = (u << 1) | br_bit(br);
        br->pos++;
      }
      z[pos] = (u & 1) == 0 ? (u >> 1) : -((u + 1) >> 1);
      pos++;
    }
  }
  return 0;
}

/* _reconstruct + _ycc_to_rgb, codec_core.py:406-411,478-489.  zz: 3 x nblocks x 64. */
static void reconstruct(const int64_t *zz, int w, int h, int quality, uint8_t *rgb) {
  int ph = (h + 7) / 8 * 8, pw = (w + 7) / 8 * 8;
  int bw_ = pw / 8;
  size_t nblocks = (size_t)(ph / 8) * bw_;
  double lqt[64], cqt[64];
  ho_quant_tables(quality, lqt, cqt);
  double *planes = malloc(sizeof(double) * 3 * (size_t)ph * pw);
  for (int ci = 0; ci < 3; ci++) {
    const double *qt = ci == 0 ? lqt : cqt;
    for (size_t bi = 0; bi < nblocks; bi++) {
      const int64_t *z = zz + ((size_t)ci * nblocks + bi) * 64;
      double coef[64], out[64];
      for (int k = 0; k < 64; k++) coef[ZIGZAG[k]] = (double)z[k] * qt[ZIGZAG[k]];
      idct8x8(coef, out);
      int by = (int)(bi / bw_), bx = (int)(bi % bw_);
      for (int yy = 0; yy < 8; yy++)
        for (int xx = 0; xx < 8; xx++)
          planes[(size_t)ci * ph * pw + (size_t)(by * 8 + yy) * pw + bx * 8 + xx] = out[yy * 8 + xx];
    }
  }
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) {
      size_t i = (size_t)y * pw + x;
      double Y = planes[i], cb = planes[(size_t)ph * pw + i], cr = planes[2 * (size_t)ph * pw + i];
      double v[3];
      v[0] = Y + 1.402 * cr;
      v[1] = Y - 0.344136 * cb - 0.714136 * cr;
      v[2] = Y + 1.772 * cb;
      for (int c = 0; c < 3; c++) {
        double r = rha(v[c]);
        r = r < 0 ? 0 : (r > 255 ? 255 : r);
        rgb[((size_t)y * w + x) * 3 + c] = (uint8_t)r;
      }
    }
  free(planes);
}

/* _BlockDctCoder.encode, codec_core.py:430-453.  sdr: (h,w,3) interleaved.
 * out: zeroed here, capacity ph*pw*3*12+1024.  decoded: (h,w,3).  zz_out
 * (optional): 3 x nblocks x 64 int64 zigzag coefficients.  Returns bits. */
uint64_t ho_lossy_encode(const uint8_t *sdr, int h, int w, int quality, uint8_t *out, uint8_t *decoded,
                         int64_t *zz_out) {
  int ph = (h + 7) / 8 * 8, pw = (w + 7) / 8 * 8;
  int nbx = pw / 8;
  size_t nblocks = (size_t)(ph / 8) * nbx;
  memset(out, 0, (size_t)ph * pw * 3 * 12 + 1024);
  double lqt[64], cqt[64];
  ho_quant_tables(quality, lqt, cqt);
  int64_t *zz = zz_out ? zz_out : malloc(sizeof(int64_t) * 3 * nblocks * 64);
  for (size_t bi = 0; bi < nblocks; bi++) {
    int by = (int)(bi / nbx), bx = (int)(bi % nbx);
    double comp[3][64];
    for (int yy = 0; yy < 8; yy++)
      for (int xx = 0; xx < 8; xx++) {
        int y = by * 8 + yy, x = bx * 8 + xx;
        if (y >= h) y = h - 1; /* np.pad mode="edge", codec_core.py:435 */
        if (x >= w) x = w - 1;
        const uint8_t *p = sdr + ((size_t)y * w + x) * 3;
        double r = p[0], g = p[1], b = p[2];
        /* _rgb_to_ycc, codec_core.py:391-403 */
        double Y = 0.299 * r + 0.587 * g + 0.114 * b;
        double cb = -0.168736 * r - 0.331264 * g + 0.5 * b;
        double cr = 0.5 * r - 0.418688 * g - 0.081312 * b;
        Y = rha(Y);
        Y = Y < 0 ? 0 : (Y > 255 ? 255 : Y);
        cb = rha(cb);
        cb = cb < -128 ? -128 : (cb > 127 ? 127 : cb);
        cr = rha(cr);
        cr = cr < -128 ? -128 : (cr > 127 ? 127 : cr);
        comp[0][yy * 8 + xx] = Y;
        comp[1][yy * 8 + xx] = cb;
        comp[2][yy * 8 + xx] = cr;
      }
    for (int ci = 0; ci < 3; ci++) {
      const double *qt = ci == 0 ? lqt : cqt;
      double coef[64];
      dct8x8(comp[ci], coef);
      int64_t *z = zz + ((size_t)ci * nblocks + bi) * 64;
      for (int k = 0; k < 64; k++) z[k] = (int64_t)rha(coef[ZIGZAG[k]] / qt[ZIGZAG[k]]);
    }
  }
  bw_t bw = {out, 0};
  int64_t A[DCT_CTX], N[DCT_CTX];
  for (int i = 0; i < DCT_CTX; i++) A[i] = 4, N[i] = 1;
  for (int ci = 0; ci < 3; ci++) encode_dct_component(&bw, zz + (size_t)ci * nblocks * 64, nblocks, ci == 0 ? 0 : 1, A, N);
  reconstruct(zz, w, h, quality, decoded);
  if (!zz_out) free(zz);
  return bw.pos;
}

/* _BlockDctCoder.decode, codec_core.py:455-476 */
int ho_lossy_decode(const uint8_t *bits, size_t nbytes, int h, int w, int quality, uint8_t *rgb) {
  int ph = (h + 7) / 8 * 8, pw = (w + 7) / 8 * 8;
  size_t nblocks = (size_t)(ph / 8) * (pw / 8);
  int64_t *zz = malloc(sizeof(int64_t) * 3 * nblocks * 64);
  br_t br = {bits, (uint64_t)nbytes * 8, 0};
  int64_t A[DCT_CTX], N[DCT_CTX];
  for (int i = 0; i < DCT_CTX; i++) A[i] = 4, N[i] = 1;
  for (int ci = 0; ci < 3; ci++) {
    int st = decode_dct_component(&br, zz + (size_t)ci * nblocks * 64, nblocks, ci == 0 ? 0 : 1, A, N);
    if (st) {
      free(zz);
      return st;
    }
  }
  reconstruct(zz, w, h, quality, rgb);
  free(zz);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Gaussian prefilter: scipy.ndimage.correlate1d, symmetric branch, mode      */
/* reflect, axis 0 then axis 1 (estimator.py:130-142).                        */
/* ------------------------------------------------------------------------- */
static inline long reflect_idx(long i, long n) {
  long m = i % (2 * n);
  if (m < 0) m += 2 * n;
  if (m >= n) m = 2 * n - 1 - m;
  return m;
}

/* taps: 2r+1 symmetric weights from numpy (gaussian_kernel, estimator.py:120-127) */
void ho_prefilter(const uint8_t *plane, int h, int w, const double *taps, int r, double *out) {
  double *tmp = malloc(sizeof(double) * (size_t)h * w);
  const double *fw = taps + r; /* centre */
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) {
      double o = (double)plane[(size_t)y * w + x] * fw[0];
      for (int jj = -r; jj < 0; jj++) {
        double lo = plane[(size_t)reflect_idx(y + jj, h) * w + x];
        double hi = plane[(size_t)reflect_idx(y - jj, h) * w + x];
        o += (lo + hi) * fw[jj];
      }
      tmp[(size_t)y * w + x] = o;
    }
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) {
      const double *row = tmp + (size_t)y * w;
      double o = row[x] * fw[0];
      for (int jj = -r; jj < 0; jj++) o += (row[reflect_idx(x + jj, w)] + row[reflect_idx(x - jj, w)]) * fw[jj];
      out[(size_t)y * w + x] = o;
    }
  free(tmp);
}

/* ------------------------------------------------------------------------- */
/* Summation order models of the reference's third-party arithmetic.          */
/* ------------------------------------------------------------------------- */

/* numpy pairwise_sum for float64 (numpy/_core/src/umath/loops_utils.h),
 * reached by x.sum() in fit_region (estimator.py:159) and by np.mean in
 * tone_map (tonemap.py:101).  Reduction initial value 0.0 + pairwise(n). */
double ho_pairwise_sum(const double *a, size_t n) {
  if (n < 8) {
    double res = 0.;
    for (size_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    size_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    size_t n2 = n / 2;
    n2 -= n2 % 8;
    return ho_pairwise_sum(a, n2) + ho_pairwise_sum(a + n2, n - n2);
  }
}

/* OpenBLAS 0.3.30 ddot compute kernels (kernel/x86_64/ddot.c + microkernels).
 * kernel 0 = SKYLAKEX (AVX-512): 32 lanes over [0,n32), fold 512->256, four
 * 4-lane accumulators over [n32,n1) in steps of 16, tail fma(y,x,dot).
 * kernel 1 = HASWELL (AVX2): 16 lanes over [0,n1), reduction per the asm
 * horizontal adds, tail dot + y*x without fma.  Both checked against
 * np.dot in tests/test_oracle.py. */
static double ddot_compute(const double *x, const double *y, size_t n, int kernel) {
  size_t n1 = n & ~(size_t)15;
  size_t i = 0;
  double dot = 0.0;
  if (kernel == 0) {
    if (n1) {
      size_t n32 = n1 & ~(size_t)31;
      double acc[32];
      for (int l = 0; l < 32; l++) acc[l] = 0.0;
      for (; i < n32; i += 32)
        for (int l = 0; l < 32; l++) acc[l] = fma(x[i + l], y[i + l], acc[l]);
      double a256[4][4];
      for (int k = 0; k < 4; k++)
        for (int l = 0; l < 4; l++) a256[k][l] = acc[8 * k + l] + acc[8 * k + l + 4];
      for (; i < n1; i += 16)
        for (int k = 0; k < 4; k++)
          for (int l = 0; l < 4; l++) a256[k][l] = fma(x[i + 4 * k + l], y[i + 4 * k + l], a256[k][l]);
      double s[4];
      for (int l = 0; l < 4; l++) s[l] = ((a256[0][l] + a256[1][l]) + a256[2][l]) + a256[3][l];
      dot = (s[0] + s[2]) + (s[1] + s[3]);
    }
    for (; i < n; i++) dot = fma(y[i], x[i], dot);
  } else {
    if (n1) {
      double acc[4][4];
      for (int k = 0; k < 4; k++)
        for (int l = 0; l < 4; l++) acc[k][l] = 0.0;
      for (; i < n1; i += 16)
        for (int k = 0; k < 4; k++)
          for (int l = 0; l < 4; l++) acc[k][l] = fma(x[i + 4 * k + l], y[i + 4 * k + l], acc[k][l]);
      double t[4][2];
      for (int k = 0; k < 4; k++) t[k][0] = acc[k][0] + acc[k][2], t[k][1] = acc[k][1] + acc[k][3];
      double u0 = t[0][0] + t[1][0], u1 = t[0][1] + t[1][1];
      double v0 = t[2][0] + t[3][0], v1 = t[2][1] + t[3][1];
      double w0 = u0 + v0, w1 = u1 + v1;
      dot = w0 + w1;
    }
    for (; i < n; i++) dot = dot + y[i] * x[i];
  }
  return dot;
}

/* ddot interface with OpenBLAS's level-1 thread split (n > 10000 and T > 1):
 * chunk = ceil(remaining / (T - used)); partials summed 0.0 + p0 + p1 + ... */
double ho_ddot(const double *x, const double *y, size_t n, int kernel, int threads) {
  if (n <= 10000 || threads <= 1) return ddot_compute(x, y, n, kernel);
  double dot = 0.0;
  size_t off = 0, rem = n;
  for (int used = 0; rem > 0; used++) {
    size_t width = (rem + (size_t)(threads - used) - 1) / (size_t)(threads - used);
    if (width > rem) width = rem;
    dot = dot + ddot_compute(x + off, y + off, width, kernel);
    off += width;
    rem -= width;
  }
  return dot;
}

/* ------------------------------------------------------------------------- */
/* SLRME fit (estimator.py:145-214) and estimate (estimator.py:217-244)       */
/* ------------------------------------------------------------------------- */

/* fit_region, estimator.py:145-169 */
static void fit_region(const double *x, const double *y, size_t n, int kernel, int threads, double *a_out,
                       double *b_out) {
  double sx = ho_pairwise_sum(x, n);
  double sy = ho_pairwise_sum(y, n);
  double sxx = 0.0 + ho_ddot(x, x, n, kernel, threads); /* numpy DOUBLE_dot: sum = 0.0 + cblas_ddot */
  double sxy = 0.0 + ho_ddot(x, y, n, kernel, threads);
  double dn = (double)n;
  double den = dn * sxx - sx * sx;
  if (den > 0.0) {
    double a = (dn * sxy - sx * sy) / den;
    double b = (sy - a * sx) / dn;
    if (isfinite(a) && isfinite(b)) {
      *a_out = a;
      *b_out = b;
      return;
    }
  }
  *a_out = 0.0;
  *b_out = sy / dn;
}

/* fit_slrme, estimator.py:172-214.  Outputs for every (channel, exponent):
 * a32[ch*256+e], b32[..] (float32), present count[e].  Returns 0 ok, or 1 when
 * some float32 parameter is non-finite (RegressionTable raises ValueError,
 * estimator.py:66-67). */
int ho_fit(const double *const sstar[3], const uint8_t *const m[3], const uint8_t *e, size_t n, int global,
           int kernel, int threads, float *a32, float *b32, uint32_t *counts) {
  size_t cnt[256] = {0};
  for (size_t i = 0; i < n; i++) cnt[e[i]]++;
  for (int k = 0; k < 256; k++) counts[k] = (uint32_t)cnt[k];
  size_t start[257];
  start[0] = 0;
  for (int k = 0; k < 256; k++) start[k + 1] = start[k] + cnt[k];
  size_t *order = malloc(sizeof(size_t) * (n ? n : 1));
  size_t fillp[256];
  memcpy(fillp, start, sizeof(fillp));
  for (size_t i = 0; i < n; i++) order[fillp[e[i]]++] = i; /* stable: raster order within a bin */
  double *xs = malloc(sizeof(double) * (n ? n : 1));
  double *ys = malloc(sizeof(double) * (n ? n : 1));
  int bad = 0;
  for (int ch = 0; ch < 3; ch++) {
    if (global) {
      for (size_t i = 0; i < n; i++) ys[i] = m[ch][i];
      double a, b;
      fit_region(sstar[ch], ys, n, kernel, threads, &a, &b);
      for (int k = 0; k < 256; k++) {
        a32[ch * 256 + k] = (float)a;
        b32[ch * 256 + k] = (float)b;
      }
      if (!isfinite((float)a) || !isfinite((float)b)) bad = 1;
      continue;
    }
    for (int k = 0; k < 256; k++) {
      a32[ch * 256 + k] = 0.0f;
      b32[ch * 256 + k] = 0.0f;
      if (!cnt[k]) continue;
      size_t nk = cnt[k];
      for (size_t j = 0; j < nk; j++) {
        size_t i = order[start[k] + j];
        xs[j] = sstar[ch][i];
        ys[j] = m[ch][i];
      }
      double a, b;
      fit_region(xs, ys, nk, kernel, threads, &a, &b);
      a32[ch * 256 + k] = (float)a; /* float(np.float32(a)): round to nearest even */
      b32[ch * 256 + k] = (float)b;
      if (!isfinite(a32[ch * 256 + k]) || !isfinite(b32[ch * 256 + k])) bad = 1;
    }
  }
  free(order);
  free(xs);
  free(ys);
  return bad;
}

/* estimate_mantissa, estimator.py:217-244: M* = clip(rha(a*S* + b), 0, 255) */
void ho_estimate(const double *sstar, const uint8_t *e, size_t n, const float *a32, const float *b32, uint8_t *out) {
  for (size_t i = 0; i < n; i++) {
    double a = a32[e[i]], b = b32[e[i]];
    double v = rha(a * sstar[i] + b);
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    out[i] = (uint8_t)v;
  }
}
