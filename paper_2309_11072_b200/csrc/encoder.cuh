// encoder.cuh -- per-image descriptor shared by every stage of the batched
// B200 encode pipeline, plus the host-side launcher declarations.
//
// One batch = a list of independent images (BASELINE configs 1 and 4).  Every
// kernel takes the device array of ImgDesc and derives its image from the
// grid (blockIdx.y) or from a flattened tile index, so a whole batch runs as
// one launch per stage.  All per-image intermediates live in one device arena
// carved by the host (api.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hdll {

struct ImgDesc {
  // geometry
  int w, h;
  long long n;          // w*h
  int pw, ph;           // padded to a multiple of 8
  int nbx, nby;         // blocks per row / column
  long long nblocks;    // nbx*nby

  // parameters (container.py:131-142)
  int quality;
  int sigma_milli;
  int slrme;
  int global_regression;
  int blas_kernel;      // 0 SKYLAKEX, 1 HASWELL
  int blas_threads;
  int radius;           // Gaussian radius ceil(3 sigma)
  int want_trace;
  double key, white_point /* <=0: auto */, inv_gamma, epsilon;
  const double* taps;   // 2*radius+1 taps computed on the host with numpy (estimator.py:120-127)
  const double* qt;     // 256 doubles: luma[64], chroma[64] (natural order), then their reciprocals

  // input
  const uint8_t* rgbe;  // (h, w, 4), 16-byte aligned
  const uint8_t* sdr_in;  // lossy-coder plugin mode: (h, w, 3) SDR given directly (codec_core.py:430)
  int crc_mask;           // which of the 5 CRC jobs to run

  // Row-band view (tile-sharded single image, api.cu band mode).  A band desc
  // is an image of the band's compute rows; these fields place it in the full
  // image.  Whole-image descs: full_n = n, pix_base = 0, every range complete.
  long long full_n;           // pixels of the full image (tone-map mean, pairwise tree)
  long long pix_base;         // full-image index of the desc's pixel 0
  long long node0, node1;     // pairwise nodes (level tm_level) this desc sums
  long long fit_p0, fit_m;    // fit samples: desc pixels [fit_p0, fit_p0 + fit_m); xs/ys plane stride
  int fit_owner;              // 1: xs/ys/bin_* were filled by the exchange (skip the sort)
  int int_fit;                // 1: sigma = 0 -- S* = S is integer, every sum exact: k_fit_int, no sort
  int hist_fused;             // 1: k_sdr_ycc builds the sort's tile histograms (whole-image fit)
  long long crc_p0, crc_np;   // CRC jobs cover desc pixels [crc_p0, crc_p0 + crc_np)

  // tone-map stage
  unsigned long long* maxlw;  // bits of max Lw (Lw >= 0)
  double* tm_nodes;           // pairwise-sum level-L node values (all 2^L of the full image)
  int tm_level;               // L for the image-wide pairwise tree
  double* scalars;            // [0] log-sum, [1] log_avg, [2] white, [3] allzero flag

  // base layer
  uint8_t* sdr;               // trace: (h, w, 3) pre-coding SDR (optional)
  uint8_t* ycc;               // 3 planes (h, w): Y u8, Cb i8, Cr i8 (rounded, clamped)
  uint8_t* s_planes;          // 3 planes (h, w): decoded S
  int16_t* zz;                // [3][nblocks][64] zigzag quantised coefficients

  // enhancement
  double* sstar;              // 3 planes (h, w) f64 (sigma > 0)
  double* sstar_tmp;          // vertical-pass scratch (h, w)
  uint8_t* e_plane;           // (h, w)
  uint8_t* res_planes;        // 3 planes (h, w)
  uint8_t* mstar;             // trace: 3 planes (optional)

  // SLRME fit
  int sort_tiles;             // tiles of kSortTile pixels
  unsigned* tile_hist;        // [256][sort_tiles] (then tile offsets)
  double* xs;                 // [3][n]: S* samples stable-sorted by E (raster order inside a bin)
  uint8_t* ys;                // [3][n]: M samples in the same order
  unsigned* bin_count;        // 256
  unsigned* bin_start;        // 257
  long long* sum_y;           // [3][256] exact integer sums of M per bin
  long long* isum;            // int_fit: [3][256][3] exact integer sums of x, x*x, x*y per bin
  double* seg_nodes;          // pairwise node values of every (channel, bin) segment
  int* seg_level;             // [3*256] L per segment
  long long* seg_node_off;    // [3*256+1] node offsets
  double* dot_part;           // [3*256][kMaxBlasThreads][2] ddot partials (xx, xy)
  float* a32;                 // [3][256]
  float* b32;                 // [3][256]

  // CRCs: 0 base (decoded RGB), 1 E, 2..4 residual R,G,B
  unsigned* crc;              // [5]
  unsigned* crc_part;         // per-chunk partial crcs
  long long crc_chunks[5];
  long long crc_part_off[5];
  long long crc_u0;           // first CRC work unit (chunk) of the image in the batch (crc_assign_units)


  // GPU decoder (decode.cu): coder bodies in, RGBE (or the SDR) out
  int decode;                 // 1: this desc decodes
  const uint8_t* pay[5];      // base, E, R, G, B coder bodies (MSB-first bits after the <II> w, h)
  long long pay_bytes[5];
  uint8_t* out_rgbe;          // (h, w, 4) decoded RGBE, or (h, w, 3) SDR for an SDR-only decode

  // output
  uint8_t* out;               // serialized stream
  unsigned long long* out_len;
  long long out_cap;
  const uint8_t* hdr_pre;     // fixed header + TMO record (host-built)
  int hdr_pre_len;
  const uint8_t* hdr_post;    // u32 length + header text block
  int hdr_post_len;
  unsigned* status;           // error bits
  unsigned* amb;              // pixels k_sdr_ycc deferred to k_sdr_fix (their fp32 pow is undecided)
  unsigned* amb_list;         // [amb_cap] their indices
  unsigned amb_cap;
};

constexpr int kMaxBlasThreads = 64;
constexpr int kSortTile = 1024;
constexpr int kCrcChunk = 1024;       // bytes per CRC partial of a plane (32 lanes x 32 bytes)
constexpr int kCrcChunkRgb = 768;     // bytes per CRC partial of the interleaved RGB job (32 lanes x 8 pixels)
constexpr int kNodeTarget = 1024;     // pairwise-sum level-L node size target

// pairwise tree level so level-L nodes hold >= kNodeTarget elements
inline __host__ __device__ int pairwise_level(long long n) {
  int L = 0;
  while ((n >> (L + 1)) >= kNodeTarget) L++;
  return L;
}

constexpr int kMaxCtx = 6;
constexpr int kDctMaxBlocksPerLane = 4;  // entropy tile: 32 lanes x ChainTab::dct_bpl consecutive blocks
constexpr int kPlaneTileRows = 32;                        // entropy tile: one row (segment) per lane

// Plane entropy tiles: a row of width w is cut into the power-of-two number of
// segments (<= 32) that brings them to at most segw samples; a tile holds
// 32 / segments rows.
__host__ __device__ inline int plane_row_segments(int w, int segw) {
  int s = 1;
  while (s < 32 && (long long)s * segw < w) s <<= 1;
  return s;
}
inline int plane_tile_rows(int w, int segw) { return kPlaneTileRows / plane_row_segments(w, segw); }

// target segment width for a launch coding `rows` plane rows in all: about
// sixteen waves of tiles over the GPU's warps, segments of >= 256 samples
inline int plane_segw_for(long long rows, int max_w) {
  // ~16 waves of tiles over the resident warps (148 SMs x 28): a tile takes
  // ~2 ms / S, and with ~2 waves the last, partial wave idles most of the GPU
  // (config 1: S = 8 measured 0.8 ms faster than S = 1; 2 and 4 in between)
#ifndef HDLL_PLANE_WAVES
#define HDLL_PLANE_WAVES 16
#endif
  const long long want_tiles = (long long)HDLL_PLANE_WAVES * 148 * 28;
  long long s = 1;
  while (s < 32 && rows * s / kPlaneTileRows < want_tiles) s <<= 1;
  int segw = (int)((max_w + s - 1) / s);
#ifndef HDLL_PLANE_MIN_SEGW
#define HDLL_PLANE_MIN_SEGW 256
#endif
  return segw < HDLL_PLANE_MIN_SEGW ? HDLL_PLANE_MIN_SEGW : segw;
}

// Sequential-coder chains for the entropy kernel (entropy.cu).
constexpr int kModeSkip = 3;  // ChainTab::chain_mode: the chain is not run

struct ChainTab {
  int nchains;
  const long long* tile_base;  // [nchains+1] global tile index of each chain's tile 0
  const int* img;              // image of the chain
  const int* kind;             // 0 = DCT stream, 1..4 = plane (E, R, G, B)
  const int* comp;             // DCT: the one component of the chain, -1 for Y, Cb, Cr in turn, -2 for Cb, Cr
  const long long* first;      // first coded unit in the image arrays (DCT block / plane row)
  const long long* units;      // coded units (DCT: blocks per component; plane: rows)
  uint8_t* const* out;         // chain byte stream (4-byte aligned)
  const long long* cap;        // capacity in bytes
  unsigned long long* bits;    // [nchains] total bits (written by the last tile)
  // A chain may continue a sequential coder run elsewhere (a row band of a
  // tile-sharded image): its first tile starts from in_cnt / in_a instead of
  // the reset state (count 0, A = 4).  mode 1 stops after the counts and
  // mode 2 after the A-maps, reporting the chain totals in out_cnt / out_map.
  const long long* in_cnt;     // [nchains][kMaxCtx] context counts before the chain
  const int* in_a;             // [nchains][kMaxCtx] A entering the chain
  long long* out_cnt;          // [nchains][kMaxCtx] counts after the chain (modes 0 and 1)
  AMap* out_map;               // [nchains][kMaxCtx] the chain's composed A-map (mode 2)
  int* out_a;                  // [nchains][kMaxCtx] A after the chain (mode 0)
  int mode;                    // 0 full encode, 1 counts, 2 counts + A-maps
  const int* chain_mode;       // [nchains] or null: per-chain mode overriding `mode` (kModeSkip: not run)
  int modes_present;           // host: bit m set when some chain runs mode m (launch_entropy_fixup)
  int plane_segw;              // plane rows are cut into segments of <= plane_segw samples
  int dct_bpl;                 // DCT chains: consecutive blocks per lane (1..kDctMaxBlocksPerLane)
  // per global tile status (epoch-tagged)
  int* flags;                  // [ntiles][4]: cnt, map, bit, done
  long long* cnt;              // [ntiles][2][kMaxCtx]: aggregate, inclusive
  AMap* maps;                  // [ntiles][kMaxCtx]: aggregate
  int* states;                 // [ntiles][kMaxCtx]: inclusive A
  unsigned long long* bitv;    // [ntiles][2]: aggregate bits, inclusive end bit
  uint32_t* edge;              // [ntiles][2]: head / tail partial words (merged by k_entropy_fixup)
  int* ticket;
  long long ntiles;
  int epoch;
  // ticket -> (chain, tile) round-robin schedule: rounds [seg_r0[k], seg_r0[k+1]) have
  // seg_active[k] chains (the first ones of rr_chain, longest first) starting at ticket seg_t0[k]
  int nseg;
  const long long* seg_r0;
  const long long* seg_t0;
  const int* seg_active;
  const int* rr_chain;
};

struct AsmTab {
  // base-layer DCT byte streams and bit totals: image i's at [i * dct_stride];
  // with dct_split its stream is that chain (Y) followed, bit-contiguously, by
  // chain [i * dct_stride + 1] (Cb, Cr)
  uint8_t* const* dct_out;
  const unsigned long long* dct_bits;
  int dct_stride = 1;
  bool dct_split = false;
  uint8_t* const* plane_out;                 // [nimg*4] E, R, G, B plane byte streams
  const unsigned long long* plane_bits;      // [nimg*4]
  unsigned* err_acc = nullptr;               // the context's accumulated status (Ctx::err_acc)
};

void upload_base_constants();
void upload_crc_constants();
void upload_fit_constants();
void upload_tonemap_constants();
void launch_tonemap_stats(const ImgDesc*, int nimg, long long max_n, int max_level, cudaStream_t);
void launch_tonemap_partial(const ImgDesc*, int nimg, long long max_n, int max_level, cudaStream_t);
void launch_tonemap_scalars(const ImgDesc*, int nimg, cudaStream_t);
void launch_base_layer(const ImgDesc*, int nimg, int max_tiles, long long max_n, cudaStream_t);
void launch_reconstruct(const ImgDesc*, int nimg, int max_tiles, cudaStream_t);
void launch_decode_coders(const ImgDesc*, int nimg, bool planes, int max_w, cudaStream_t);
void launch_decode_output(const ImgDesc*, int nimg, long long max_n, cudaStream_t);
void launch_hdr_sizes(const uint8_t* rgbe, int w, int h, long long* sizes, cudaStream_t);
void launch_hdr_write(const uint8_t* rgbe, int w, int h, const long long* offs, uint8_t* out, cudaStream_t);
void launch_hdr_expand(const uint8_t* data, const long long* starts, const uint8_t* newrle, int w, int h, uint8_t* rgbe,
                       cudaStream_t);
// any_non3: some image of the batch filters with a radius other than 3 (else the
// general kernels are not launched at all)
void launch_prefilter(const ImgDesc*, int nimg, int max_w, int max_h, int max_radius, cudaStream_t, bool any_non3 = true);
// any_hist: some image needs k_sort_hist (its histogram is not fused into k_sdr_ycc)
void launch_fit(const ImgDesc*, int nimg, int max_sort_tiles, long long max_nodes, int max_chunks, cudaStream_t,
                bool any_hist = true);
void launch_fit_sort(const ImgDesc*, int nimg, int max_sort_tiles, cudaStream_t, bool any_hist = true);
void launch_fit_bins(const ImgDesc*, int nimg, long long max_nodes, int max_chunks, cudaStream_t);
void launch_fit_int(const ImgDesc*, int nimg, long long max_n, cudaStream_t);
void launch_fit_int_sums(const ImgDesc*, int nimg, long long max_n, cudaStream_t);
void launch_fit_int_coef(const ImgDesc*, int nimg, cudaStream_t);
void launch_fit_hist(const ImgDesc*, int nimg, int max_sort_tiles, cudaStream_t);
struct RegroupTab {
  int nsrc;
  const uint8_t* recv;             // concatenated chunks, one per source rank
  const long long* src_off;        // [nsrc+1] byte offset of each chunk
  const long long* src_m;          // [nsrc] samples in each chunk
  const unsigned* src_bin_off;     // [nsrc][257] sample offset of bin e inside the chunk (owned bins)
  const unsigned* dst_bin_off;     // [nsrc][256] destination of the chunk's first sample of bin e
  long long total;                 // samples received
};
void launch_fit_regroup(const ImgDesc* d, const RegroupTab&, cudaStream_t);
void launch_bitcat(uint8_t* dst, const uint8_t* const* src, const unsigned long long* dst_bit, const unsigned long long* nbits,
                   int npieces, unsigned long long max_bits, cudaStream_t);
void launch_estimate(const ImgDesc*, int nimg, long long max_n, cudaStream_t);
// CRC chunks of the batch's active jobs, numbered image by image: sets each
// descriptor's crc_u0 (after crc_mask / crc_np are final) and returns the total
long long crc_assign_units(ImgDesc* ds, int n);
void launch_crc(const ImgDesc*, int nimg, long long units, cudaStream_t);
// both coders keep per-warp scratch in one device buffer (they run one after the other)
size_t dct_scratch_bytes(const ChainTab&);
void launch_entropy_dct(const ImgDesc*, const ChainTab&, void* scratch, cudaStream_t);
size_t plane_scratch_bytes(const ChainTab&, int max_w);
void launch_entropy_plane(const ImgDesc*, const ChainTab&, int max_w, void* scratch, cudaStream_t);
void launch_entropy_fixup(const ChainTab&, cudaStream_t);
void launch_assemble(const ImgDesc*, int nimg, const AsmTab&, long long max_out, cudaStream_t);

}  // namespace hdll
