/*
 * hdll_b200.h -- C ABI of the B200-native hdll encoder hot path.
 *
 * Drop-in boundary for the reference package `hdll` (/root/reference/pkg).
 * The reference is pure Python, so "its FFI" for this path is a ctypes
 * binding; each entry point below replaces one reference interface:
 *
 *   hdll_b200_encode_batch_device / hdll_b200_encode_host
 *       replace hdll.container.encode (container.py:131-230) followed by
 *       serialize (container.py:332-340): RGBE quads in, the serialized HDLL v1
 *       stream out (byte-identical to the reference's).
 *   hdll_b200_lossless_encode_plane
 *       replaces the lossless coder plugin id 1 `_MedRicePlaneCoder.encode`
 *       (codec_core.py:260-265) plus the CRC of lossless_encode (:306-313).
 *   hdll_b200_lossy_encode
 *       replaces the lossy coder plugin id 1 `_BlockDctCoder.encode`
 *       (codec_core.py:430-453) plus the CRC of lossy_encode (:520-533).
 *
 * Plain pointers and sizes only.  Device pointers are CUDA global memory;
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Status codes are
 * mapped to the reference's Python exceptions by paper_2309_11072_b200/_native.py.
 */
#ifndef HDLL_B200_H
#define HDLL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdll_b200_ctx hdll_b200_ctx;

enum {
  HDLL_B200_OK = 0,
  HDLL_B200_E_ARG = 1,          /* bad argument (ValueError in the reference) */
  HDLL_B200_E_EMPTY = 2,        /* empty image (StreamError, container.py:154-155) */
  HDLL_B200_E_NONFINITE = 3,    /* float32 a/b overflow (ValueError, estimator.py:66-67) */
  HDLL_B200_E_CUDA = 4,         /* CUDA runtime error */
  HDLL_B200_E_INTERNAL = 5,     /* device-side consistency failure */
  HDLL_B200_E_CAPACITY = 6      /* output buffer too small */
};

/* Encode parameters (container.py:131-142, TmoParams tonemap.py:22-37). */
typedef struct hdll_b200_params {
  int32_t quality;           /* 1..100 */
  int32_t sigma_milli;       /* round(sigma * 1000), 0 = no prefilter */
  int32_t slrme;             /* 0/1 */
  int32_t global_regression; /* 0/1 */
  int32_t blas_kernel;       /* sum-order model of np.dot: 0 OpenBLAS SKYLAKEX, 1 HASWELL */
  int32_t blas_threads;      /* OpenBLAS thread count of the modelled reference run (>= 1) */
  int32_t radius;            /* Gaussian radius ceil(3 sigma) */
  int32_t want_trace;        /* keep sdr / s / m_star / residual planes for hdll_b200_trace */
  double tmo_key;
  double tmo_white_point;    /* <= 0: automatic (max of the scaled luminance) */
  double tmo_inv_gamma;      /* 1.0 / gamma as the host computes it */
  double tmo_epsilon;
  const double *taps;        /* host pointer, 2*radius+1 Gaussian taps (numpy gaussian_kernel) */
} hdll_b200_params;

typedef struct hdll_b200_image {
  const uint8_t *rgbe;       /* (height, width, 4) RGBE quads; device or host pointer per call */
  uint32_t width, height;
  const uint8_t *hdr_pre;    /* host bytes: magic .. sigma_milli + u16 len + TMO record */
  uint32_t hdr_pre_len;
  const uint8_t *hdr_post;   /* host bytes: u32 len + header text block */
  uint32_t hdr_post_len;
  hdll_b200_params params;
} hdll_b200_image;

int hdll_b200_ctx_create(hdll_b200_ctx **out, int device);
void hdll_b200_ctx_destroy(hdll_b200_ctx *ctx);

/* Upper bound of the serialized stream length for one image. */
uint64_t hdll_b200_stream_capacity(uint32_t width, uint32_t height, uint32_t hdr_pre_len, uint32_t hdr_post_len);

/* Batched encode, everything resident on the device.  d_out[i] receives image
 * i's stream (capacity out_cap[i] bytes), d_out_len[i] its length, written
 * by a kernel: device memory, or pinned host memory (mapped under unified
 * addressing), which then holds the lengths once `stream` has reached the end
 * of the batch, without a device-to-host copy.
 * Asynchronous on `stream`; hdll_b200_sync() reports device-side errors. */
int hdll_b200_encode_batch_device(hdll_b200_ctx *ctx, const hdll_b200_image *imgs, int n, uint8_t *const *d_out,
                                  const uint64_t *out_cap, uint64_t *d_out_len, void *stream);

/* Wait for the last batch of this context and return the worst status of
 * every encode batch since the previous sync (device errors of earlier batches
 * of a pipeline are accumulated on the device, not lost). */
int hdll_b200_sync(hdll_b200_ctx *ctx);

/* Host -> host convenience: H2D of the RGBE quads, encode, D2H of the stream. */
int hdll_b200_encode_host(hdll_b200_ctx *ctx, const hdll_b200_image *img, uint8_t *h_out, uint64_t cap,
                          uint64_t *out_len);

/* Per-stage trace of image `index` of the last batch (want_trace set):
 * which = 0 sdr (h,w,3), 1 decoded S (h,w,3 interleaved), 2 m_star (3 planes),
 * 3 residuals (3 planes).  which | 16: the same arrays (1 and 3 only) of the
 * last hdll_b200_decode_batch (the decode_hdr trace hook, container.py:269-271).
 * nbytes must equal the array size. */
int hdll_b200_trace(hdll_b200_ctx *ctx, int index, int which, uint8_t *h_dst, uint64_t nbytes);

/* Lossless coder id 1 body (<II w,h> + bits) and the raw-plane CRC-32. */
int hdll_b200_lossless_encode_plane(hdll_b200_ctx *ctx, const uint8_t *h_plane, uint32_t width, uint32_t height,
                                    uint8_t *h_body, uint64_t cap, uint64_t *body_len, uint32_t *crc);

/* Lossy coder id 1 body, the decoded image (h,w,3) and the CRC of its bytes. */
int hdll_b200_lossy_encode(hdll_b200_ctx *ctx, const uint8_t *h_rgb, uint32_t width, uint32_t height,
                           int32_t quality, uint8_t *h_body, uint64_t cap, uint64_t *body_len, uint8_t *h_decoded,
                           uint32_t *crc);

/* Number of kernel launches issued by the last encode call. */
int hdll_b200_last_launch_count(hdll_b200_ctx *ctx);

/* Device time (ms) of the 9 stages of the last batch, in order: tonemap stats,
 * base layer, prefilter, fit, estimate, crc, DCT entropy coder, plane entropy
 * coders, assemble. */
int hdll_b200_stage_times(hdll_b200_ctx *ctx, float *ms, int n);

const char *hdll_b200_status_string(int status);

/* ---------------------------------------------------------------------------
 * GPU decoder: decode_hdr / decode_sdr (container.py:233-280),
 * lossy_decode (codec_core.py:536-548), lossless_decode (:316-331).  The host
 * parses the stream (header, table, frames); the coder bodies (after their
 * <II> w, h) go to the device, the adaptive-Rice streams are decoded one
 * thread per stream, the rest runs data parallel.
 * ------------------------------------------------------------------------- */
typedef struct hdll_b200_decode_image {
  uint32_t width, height;
  int32_t quality, slrme, sigma_milli, radius;
  int32_t sdr_only;          /* 1: decode_sdr -- base layer only, output (h, w, 3);
                                2: body[1] alone as a lossless plane (coder plugin decode), output (h, w) */
  const double *taps;        /* host, 2 * radius + 1 Gaussian taps (sigma_milli > 0) */
  const float *a32, *b32;    /* host [3][256] regression table, absent entries NaN */
  const uint8_t *body[5];    /* host: base, E, R, G, B coder bodies without their <II> w, h */
  uint64_t body_len[5];
  uint32_t crc[5];           /* the frames' CRC-32 fields */
} hdll_b200_decode_image;

enum {
  HDLL_B200_DEC_BAD = 1 << 0,        /* bit k: coder body k ended early or is inconsistent (CorruptPayloadError) */
  HDLL_B200_DEC_CRC = 1 << 8,        /* bit 8 + k: payload k failed its CRC-32 (ChecksumError) */
  HDLL_B200_DEC_NO_ENTRY = 1 << 13   /* an exponent has no regression entry (StreamError) */
};

/* Decode a batch; d_out[i] (device) receives image i's (h, w, 4) RGBE quads
 * (or (h, w, 3) SDR), h_status[i] its decode status bits (0 = ok).  Returns
 * after the batch completes. */
int hdll_b200_decode_batch(hdll_b200_ctx *ctx, const hdll_b200_decode_image *imgs, int n, uint8_t *const *d_out,
                           uint32_t *h_status, void *stream);

/* ---------------------------------------------------------------------------
 * Radiance .hdr scanlines (radiance_io.py:119-317).  The host
 * parses the text header and resolution line; these code the binary part.
 * ------------------------------------------------------------------------- */
enum {  /* scanline format errors (RadianceFormatError in the reference) */
  HDLL_B200_HDR_LENGTH = 16,        /* new-RLE scanline length != width (detail: length, width) */
  HDLL_B200_HDR_TRUNC_LINE = 17,    /* truncated new-RLE scanline */
  HDLL_B200_HDR_TRUNC_RUN = 18,     /* truncated new-RLE run */
  HDLL_B200_HDR_RUN_OVERFLOW = 19,  /* RLE run overflows scanline width */
  HDLL_B200_HDR_ZERO_LITERAL = 20,  /* zero-length literal packet */
  HDLL_B200_HDR_LIT_OVERFLOW = 21,  /* RLE literal overflows scanline width */
  HDLL_B200_HDR_TRUNC_LIT = 22,     /* truncated new-RLE literal */
  HDLL_B200_HDR_TRUNC_DATA = 23,    /* truncated scanline data (flat / old-RLE) */
  HDLL_B200_HDR_REPEAT_FIRST = 24,  /* repeat marker before any pixel */
  HDLL_B200_HDR_REPEAT_OVERFLOW = 25 /* old-RLE repeat overflows scanline width */
};

/* Scanline bytes (everything after the resolution line) -> d_rgbe (h, w, 4)
 * on the device.  h_consumed: bytes used; h_detail[2]: values for the message. */
int hdll_b200_hdr_decode(hdll_b200_ctx *ctx, const uint8_t *h_data, uint64_t len, uint32_t width, uint32_t height,
                         uint8_t *d_rgbe, uint64_t *h_consumed, int64_t *h_detail, void *stream);
/* d_rgbe (h, w, 4) on the device -> scanline bytes on the host (new-RLE for
 * widths 8..32767 when rle, else flat).  Capacity: 4 h (1 + w + (w + 127) / 128) + 4 h w suffices. */
int hdll_b200_hdr_encode(hdll_b200_ctx *ctx, const uint8_t *d_rgbe, uint32_t width, uint32_t height, int32_t rle,
                         uint8_t *h_out, uint64_t cap, uint64_t *h_len, void *stream);

/* ---------------------------------------------------------------------------
 * Tile-sharded single image (BASELINE config 3).  The reference
 * encodes one image in one process (container.py:131-230); here each rank of
 * a job codes a contiguous band of rows and the ranks exchange only the
 * summaries the sequential stages need.  The phases below run in order on
 * every rank; between them the host exchanges the named outputs (allgather,
 * all-to-all) and passes the combined values to the next phase.  Each phase
 * returns once its host outputs are ready.  Per rank, pieces 0..2 are the
 * Y, Cb, Cr slices of the base-layer DCT stream and 3..6 the E, R, G, B plane
 * streams; a chain's pieces are ordered by rank (DCT: component, then rank).
 * ------------------------------------------------------------------------- */
typedef struct hdll_b200_band {
  uint32_t row0, row1;    /* rows coded by this rank; row0 % 8 == 0, row1 % 8 == 0 or row1 == height */
  uint32_t crow0, crow1;  /* rows present at image.rgbe: the band plus halo, crow0 % 8 == 0 */
  uint64_t node0, node1;  /* level-L pairwise nodes of the tone-map log sum this rank computes */
} hdll_b200_band;

enum { HDLL_B200_BAND_PIECES = 7, HDLL_B200_BAND_CTX = 6 };

/* Phase 1.  img: full-image width/height/params; img->rgbe = device pointer to
 * rows [crow0, crow1).  Out: the rank's node sums (node1 - node0 doubles) and
 * its max luminance.  Exchange: allgather nodes (concatenate), max of maxlw. */
int hdll_b200_band_begin(hdll_b200_ctx *ctx, const hdll_b200_image *img, const hdll_b200_band *band, void *stream,
                         double *h_nodes, double *h_maxlw);
/* Phase 2: tone-map scalars from all 2^L nodes, base layer, prefilter, sort of
 * the band's fit samples by exponent.  Out: the band's exponent histogram. */
int hdll_b200_band_layers(hdll_b200_ctx *ctx, const double *h_nodes_all, uint64_t n_nodes, double maxlw,
                          uint32_t *h_hist);
/* Phases 3-4 for sigma = 0 (S* = S: every regression sum is an exact integer).
 * fit_sums: the band's table, int64 [3][256][3] sums of x, x^2, x*y then
 * [3][256] sums of y (3072 values, 24 KB).  Exchange: all-reduce (sum) of the
 * tables and of the histograms.  fit_coef: the coefficients from the summed
 * table and histogram -- identical on every rank, no sample crosses ranks.
 * Out: a32/b32 [3][256], error bits. */
int hdll_b200_band_fit_sums(hdll_b200_ctx *ctx, int64_t *h_sums);
int hdll_b200_band_fit_coef(hdll_b200_ctx *ctx, const int64_t *h_sums, const uint32_t *h_hist, float *h_a32,
                            float *h_b32, uint32_t *h_status);
/* Phases 3-4 on a single rank (the band is the whole image): fit from the
 * band's own sorted samples, no exchange.  Out: a32/b32 [3][256], error bits. */
int hdll_b200_band_fit_local(hdll_b200_ctx *ctx, float *h_a32, float *h_b32, uint32_t *h_status);
/* Phase 3: pack the sorted samples for their owners (owner o fits exponents
 * [owner_lo[o], owner_lo[o+1])) into d_send; h_send_bytes[o] = chunk sizes.
 * Exchange: all-to-all of the chunks. */
int hdll_b200_band_fit_send(hdll_b200_ctx *ctx, const uint32_t *owner_lo, int nowners, uint8_t *d_send,
                            uint64_t send_cap, uint64_t *h_send_bytes);
/* Phase 4 (owner): fit exponents [e_lo, e_hi) from the received chunks (one per
 * source rank, h_hist = every source's histogram).  Out: a32/b32 [3][256]
 * (owned entries), error bits.  Exchange: allgather of the tables. */
int hdll_b200_band_fit_owner(hdll_b200_ctx *ctx, const uint8_t *d_recv, const uint64_t *h_recv_bytes,
                             const uint32_t *h_hist, int nsrc, uint32_t e_lo, uint32_t e_hi, float *h_a32,
                             float *h_b32, uint32_t *h_status);
/* Phase 5: estimate with the full table, CRCs of the band's rows, and a coder
 * pass over the pieces.  A piece with h_first[k] set starts its chain (the
 * first rank's Y, Cb and plane pieces: nothing enters them) and is coded now
 * from the reset state -- its outgoing A h_out_a[k][6] (the next piece's
 * entering A, no map of it needed), bit length h_bits[k] and stream are final;
 * the other pieces are only counted.  Out: crc[5], counts [7][6] of every
 * piece, piece stream addresses (valid until the next begin).
 * Exchange: allgather counts (and the first pieces' outgoing A). */
int hdll_b200_band_code(hdll_b200_ctx *ctx, const float *h_a32, const float *h_b32, const int32_t *h_first,
                        uint32_t *h_crc, int64_t *h_cnt, int32_t *h_out_a, uint64_t *h_bits, uint64_t *h_piece_ptr);
/* Phase 6: A-maps of the pieces with h_need[k] set (a later piece of the chain
 * composes them; not the chain's first or last piece) given the counts before
 * them.  Out: [7][6][3] (c, s, t of common.cuh AMap).  Exchange: allgather
 * maps (skipped when no rank needs one). */
int hdll_b200_band_maps(hdll_b200_ctx *ctx, const int64_t *h_in_cnt, const int32_t *h_need, int64_t *h_maps);
/* Phase 7: code the pieces with h_emit[k] set (those not coded in phase 5)
 * given their entering counts and A.  Out: bit lengths [7] (emitted pieces)
 * and the device addresses of the piece streams. */
int hdll_b200_band_emit(hdll_b200_ctx *ctx, const int64_t *h_in_cnt, const int32_t *h_in_a, const int32_t *h_emit,
                        uint64_t *h_bits, uint64_t *h_piece_ptr);
/* Rank 0: concatenate the pieces of the 5 chains (npieces[k] each, in order;
 * piece_ptr device addresses, piece_bits lengths) and serialize the stream
 * with the combined CRCs, table and full-image exponent histogram. */
int hdll_b200_assemble_pieces(hdll_b200_ctx *ctx, const hdll_b200_image *img, const uint32_t *crc,
                              const float *a32, const float *b32, const uint32_t *hist, const int32_t *npieces,
                              const uint64_t *piece_ptr, const uint64_t *piece_bits, uint8_t *d_out, uint64_t cap,
                              uint64_t *d_len, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HDLL_B200_H */
