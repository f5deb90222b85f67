// host_common.cuh -- host-side helpers shared by the batch encoder (api.cu)
// and the row-band encoder for tile-sharded images (band.cu): the device
// context, arena layout, descriptor filling and the entropy chain tables.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/hdll_b200.h"
#include "encoder.cuh"

namespace hdll_host {
struct Band;
}

namespace hdll_host {
using namespace hdll;

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// quantization_tables (codec_core.py:375-388)
inline void quant_tables(int quality, double* out128) {
  static const double luma[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                                  14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                                  18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                                  49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
  static const double chroma[64] = {17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99,
                                    24, 26, 56, 99, 99, 99, 99, 99, 47, 66, 99, 99, 99, 99, 99, 99,
                                    99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99,
                                    99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99};
  volatile double scale = quality < 50 ? 5000.0 / quality : 200.0 - 2.0 * quality;
  for (int i = 0; i < 64; i++) {
    volatile double t = luma[i] * scale;
    t = t / 100.0;
    double r = std::trunc(t + std::copysign(0.5, (double)t));
    out128[i] = r < 1 ? 1 : (r > 255 ? 255 : r);
    t = chroma[i] * scale;
    t = t / 100.0;
    r = std::trunc(t + std::copysign(0.5, (double)t));
    out128[64 + i] = r < 1 ? 1 : (r > 255 ? 255 : r);
  }
}

// a block's code <= 544 bytes; the buffer holds the Y chain, then the Cb, Cr chain
inline long long dct_y_cap(long long nblocks) { return (nblocks * 544 + 64 + 15) / 16 * 16; }
inline long long dct_chain_cap(long long nblocks) { return dct_y_cap(nblocks) + (2 * nblocks * 544 + 64 + 15) / 16 * 16; }
inline long long plane_chain_cap(long long n) { return (n * 8 + 64 + 15) / 16 * 16; }
inline long long max_seg_nodes(long long n) { return 3 * (2 * (n / kNodeTarget) + 2 * 256 + 2); }

struct ImgLayout {
  size_t off_qt, off_taps, off_pre, off_post;
  size_t off_tmnodes, off_scalars;
  size_t off_sdr, off_ycc, off_s, off_zz;
  size_t off_sstar, off_sstar_tmp, off_e, off_res, off_mstar, off_amb;
  size_t off_tile_hist, off_xs, off_ys, off_bin_start, off_seg_nodes, off_seg_level, off_seg_node_off, off_dot, off_a32,
      off_b32;
  size_t off_crc, off_crc_part;
  size_t off_chain[5];
  long long chain_cap[5];
  size_t off_zero;  // small zero-initialised block: maxlw, status, bin_count, sum_y
  size_t total;
};

// stage boundaries recorded with CUDA events (hdll_b200_stage_times)
enum { kStTonemap, kStBase, kStPrefilter, kStFit, kStEstimate, kStCrc, kStEntropyDct, kStEntropyPlane, kStAssemble,
       kStages };

constexpr size_t kEstatPerTile = 16 + 16 * kMaxCtx + sizeof(AMap) * kMaxCtx + 4 * kMaxCtx + 16 + 8;

constexpr size_t kZeroBytes = 8 /*maxlw*/ + 8 /*status, amb*/ + 1024 /*bin_count*/ + 8 * 768 /*sum_y*/ +
                              8 * 3 * 768 /*isum*/;

struct Ctx {
  // Every C entry point taking the context holds this lock (CtxLock), so
  // threads sharing a context serialise instead of racing on the arena, the
  // staging slots and the entropy status; a batch launched on another stream
  // than the previous one waits for it on the device (run_batch).
  std::recursive_mutex mu;
  int device = 0;
  // device-side OR of every encode batch's image status words since the last
  // hdll_b200_sync (k_assemble folds each image's word in), so an error in an
  // earlier batch of a pipeline is not lost when a later batch reuses the
  // descriptors
  unsigned* err_acc = nullptr;
  void* arena = nullptr;
  size_t arena_cap = 0;
  // entropy status (epoch-tagged, zeroed once at allocation)
  void* estat = nullptr;
  long long estat_tiles = 0;
  int epoch = 0;
  // small per-batch device tables and their pinned host staging, double-buffered
  // so the host prepares batch k+1 while batch k runs
  void* tabs_slot[2] = {nullptr, nullptr};
  size_t tabs_cap_slot[2] = {0, 0};
  void* pinned_slot[2] = {nullptr, nullptr};
  size_t pinned_cap_slot[2] = {0, 0};
  cudaEvent_t slot_ev[2] = {nullptr, nullptr};
  int slot = 0;
  void* tabs = nullptr;  // slot of the last batch
  cudaEvent_t done_ev = nullptr;
  cudaEvent_t stage_ev[kStages + 1] = {};
  bool stage_valid[kStages] = {};
  cudaStream_t last_stream = nullptr;
  int launches = 0;
  int last_status = 0;
  size_t bits_off_dct = 0, bits_off_pln = 0;  // device offsets (in tabs) of the chain bit totals
  // last batch (for traces / status)
  std::vector<ImgDesc> descs;
  std::vector<ImgLayout> lays;
  std::vector<ImgDesc> dec_descs;  // last decode batch (hdll_b200_trace, which | 16)
  ImgDesc* d_descs = nullptr;
  // scratch for the host convenience path
  void* h2d = nullptr;
  size_t h2d_cap = 0;
  uint8_t* d_out = nullptr;
  size_t d_out_cap = 0;
  uint64_t* d_len = nullptr;
  Band* band = nullptr;  // row-band session (band.cu)
  void* plane_scratch = nullptr;  // plane coder symbol slabs (entropy.cu)
  size_t plane_scratch_cap = 0;
  void* hdr_buf = nullptr;  // .hdr scanline coding (hdrio.cu)
  size_t hdr_cap = 0;
};

inline int cuda_fail(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fprintf(stderr, "hdll_b200: %s: %s\n", what, cudaGetErrorString(e));
    return HDLL_B200_E_CUDA;
  }
  return HDLL_B200_OK;
}
struct CtxLock {
  std::unique_lock<std::recursive_mutex> g;
  explicit CtxLock(Ctx* c) {
    if (c) g = std::unique_lock<std::recursive_mutex>(c->mu);
  }
};

#define CK(x)                                      \
  do {                                             \
    int _rc = cuda_fail((x), #x);                  \
    if (_rc) return _rc;                           \
  } while (0)

inline int ensure(void** p, size_t* cap, size_t need, bool device, bool zero = false) {
  if (*cap >= need && *p) return 0;
  if (*p) {
    if (device) cudaFree(*p); else cudaFreeHost(*p);
    *p = nullptr;
  }
  size_t sz = need + need / 4 + (1 << 20);
  if (device) {
    CK(cudaMalloc(p, sz));
    if (zero) CK(cudaMemset(*p, 0, sz));
  } else {
    CK(cudaMallocHost(p, sz));
  }
  *cap = sz;
  return 0;
}

// tone-map pixels k_sdr_ycc may defer to k_sdr_fix (~0.3 % occur; beyond the
// cap they are decided in place)
inline long long amb_cap(long long n) { return n / 32 + 1024; }

inline ImgLayout plan(const hdll_b200_image& im, bool trace) {
  ImgLayout L{};
  const long long w = im.width, h = im.height, n = w * h;
  const long long nb = ((w + 7) / 8) * ((h + 7) / 8);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  L.off_zero = take(kZeroBytes);
  L.off_qt = take(256 * sizeof(double));
  L.off_taps = take(sizeof(double) * (2 * (size_t)std::max(0, im.params.radius) + 1));
  L.off_pre = take(im.hdr_pre_len + 1);
  L.off_post = take(im.hdr_post_len + 1);
  L.off_tmnodes = take(sizeof(double) * ((size_t)1 << pairwise_level(n)));
  L.off_scalars = take(sizeof(double) * 4);
  L.off_sdr = trace ? take(3 * n) : 0;
  L.off_ycc = take(3 * n + 16);
  L.off_s = take(3 * n + 16);
  L.off_zz = take(sizeof(int16_t) * 3 * nb * 64);
  const bool real = im.params.slrme && im.params.sigma_milli != 0;
  L.off_sstar = real ? take(sizeof(double) * 3 * n) : 0;
  L.off_sstar_tmp = real ? take(sizeof(double) * 3 * n) : 0;
  L.off_e = take(n + 16);
  L.off_amb = take(sizeof(unsigned) * (size_t)amb_cap(n));
  L.off_res = take(3 * n + 16);
  L.off_mstar = trace ? take(3 * n) : 0;
  const long long sort_tiles = (n + kSortTile - 1) / kSortTile;
  L.off_tile_hist = take(sizeof(unsigned) * 256 * sort_tiles);
  L.off_xs = take(sizeof(double) * 3 * n);
  L.off_ys = take(3 * n + 16);
  L.off_bin_start = take(sizeof(unsigned) * 257);
  L.off_seg_nodes = take(sizeof(double) * max_seg_nodes(n));
  L.off_seg_level = take(sizeof(int) * 768);
  L.off_seg_node_off = take(sizeof(long long) * 769);
  L.off_dot = take(sizeof(double) * 768 * kMaxBlasThreads * 2);
  L.off_a32 = take(sizeof(float) * 768);
  L.off_b32 = take(sizeof(float) * 768);
  L.off_crc = take(sizeof(unsigned) * 8);
  L.off_crc_part = take(sizeof(unsigned) * ((3 * n + kCrcChunkRgb - 1) / kCrcChunkRgb + 4 * ((n + kCrcChunk - 1) / kCrcChunk) + 8));
  L.chain_cap[0] = dct_chain_cap(nb);
  for (int k = 1; k < 5; k++) L.chain_cap[k] = plane_chain_cap(n);
  for (int k = 0; k < 5; k++) L.off_chain[k] = take(L.chain_cap[k]);
  L.total = o;
  return L;
}

inline int map_status(unsigned bits) {
  if (bits & kErrNonFinite) return HDLL_B200_E_NONFINITE;
  if (bits & kErrCapacity) return HDLL_B200_E_CAPACITY;
  if (bits & (kErrLookback | kErrInternal)) return HDLL_B200_E_INTERNAL;
  return HDLL_B200_OK;
}

// Host side of a ChainTab: chains, their tiles and the round-robin ticket schedule.
struct HostChains {
  std::vector<long long> tile_base{0};
  std::vector<int> img, kind, comp;
  std::vector<long long> first, units;
  std::vector<uint8_t*> out;
  std::vector<long long> cap;
  std::vector<long long> in_cnt;  // [chain][kMaxCtx]
  std::vector<int> in_a;          // [chain][kMaxCtx]
  std::vector<int> rr_chain;
  std::vector<long long> seg_r0, seg_t0;
  std::vector<int> seg_active;

  // chain of image i, kind k over `units` blocks / rows from `first`, DCT component cp (-1: all three);
  // plane tiles hold plane_tile_rows(width) rows
  int segw = 1 << 30;  // plane segment width (set before adding plane chains)
  int dct_bpl = 1;     // DCT blocks per lane (set before adding DCT chains)
  void add(int i, int k, int cp, long long fst, long long nunits, uint8_t* o, long long c, int width) {
    img.push_back(i);
    kind.push_back(k);
    comp.push_back(cp);
    first.push_back(fst);
    units.push_back(nunits);
    out.push_back(o);
    cap.push_back(c);
    for (int q = 0; q < kMaxCtx; q++) {
      in_cnt.push_back(0);
      in_a.push_back(4);  // AdaptiveRiceState: A = 4 (_kernels.py:114-128)
    }
    const long long per = k == 0 ? 32LL * dct_bpl : plane_tile_rows(width, segw);
    const long long tiles = (k == 0 && cp < 0 ? (cp == -2 ? 2 : 3) : 1) * ((nunits + per - 1) / per);
    tile_base.push_back(tile_base.back() + tiles);
  }
  int nchains() const { return (int)img.size(); }
  long long ntiles() const { return tile_base.back(); }
  long long len(int ch) const { return tile_base[ch + 1] - tile_base[ch]; }
  // chains sorted longest first; segment k spans the rounds in which exactly
  // seg_active[k] chains still have tiles; ticket t of a segment is chain
  // rr_chain[(t - t0) % active], tile r0 + (t - t0) / active
  void schedule() {
    for (int ch = 0; ch < nchains(); ch++)
      if (len(ch) > 0) rr_chain.push_back(ch);
    std::stable_sort(rr_chain.begin(), rr_chain.end(), [&](int a, int b) { return len(a) > len(b); });
    long long r = 0, t = 0;
    for (int act = (int)rr_chain.size(); act > 0; act--) {
      long long l = len(rr_chain[act - 1]);
      if (l > r) {
        seg_r0.push_back(r);
        seg_t0.push_back(t);
        seg_active.push_back(act);
        t += (l - r) * act;
        r = l;
      }
    }
    if (seg_r0.empty()) {
      seg_r0.push_back(0);
      seg_t0.push_back(0);
      seg_active.push_back(1);
    }
    if (rr_chain.empty()) rr_chain.push_back(0);
    if (img.empty()) add(0, 1, -1, 0, 0, nullptr, 0, 1);  // keep device arrays non-empty
  }
  size_t staged_bytes() const {
    size_t nc = img.size() + 2;
    return 17 * kAlign + 8 * (nc + 1) + 4 * nc * 3 + 8 * nc * 5 + (8 + 4 + 8 + 4 + sizeof(AMap)) * kMaxCtx * nc +
           8 * 2 * seg_r0.size() + 4 * seg_active.size() + 4 * rr_chain.size();
  }
  struct Staged {
    size_t tile_base, img, kind, comp, first, units, out, cap, bits, in_cnt, in_a, out_cnt, out_map, out_a, seg_r0, seg_t0,
        seg_active, rr_chain;
  };
  template <class F>
  Staged stage(F& st) const {
    Staged s;
    const size_t nc = img.size();
    s.tile_base = st(tile_base.data(), 8 * tile_base.size());
    s.img = st(img.data(), 4 * nc);
    s.kind = st(kind.data(), 4 * nc);
    s.comp = st(comp.data(), 4 * nc);
    s.first = st(first.data(), 8 * nc);
    s.units = st(units.data(), 8 * nc);
    s.out = st(out.data(), 8 * nc);
    s.cap = st(cap.data(), 8 * nc);
    s.bits = st(nullptr, 8 * nc);
    s.in_cnt = st(in_cnt.data(), 8 * in_cnt.size());
    s.in_a = st(in_a.data(), 4 * in_a.size());
    s.out_cnt = st(nullptr, 8 * kMaxCtx * nc);
    s.out_map = st(nullptr, sizeof(AMap) * kMaxCtx * nc);
    s.out_a = st(nullptr, 4 * kMaxCtx * nc);
    s.seg_r0 = st(seg_r0.data(), 8 * seg_r0.size());
    s.seg_t0 = st(seg_t0.data(), 8 * seg_t0.size());
    s.seg_active = st(seg_active.data(), 4 * seg_active.size());
    s.rr_chain = st(rr_chain.data(), 4 * rr_chain.size());
    return s;
  }
  // status arrays live in the shared entropy arena at tile offset `t0`
  ChainTab table(const Staged& s, uint8_t* D, uint8_t* E, long long cap_t, long long t0, int* ticket, int epoch,
                 int mode = 0) const {
    ChainTab ct;
    ct.nchains = nchains();
    ct.tile_base = (const long long*)(D + s.tile_base);
    ct.img = (const int*)(D + s.img);
    ct.kind = (const int*)(D + s.kind);
    ct.comp = (const int*)(D + s.comp);
    ct.first = (const long long*)(D + s.first);
    ct.units = (const long long*)(D + s.units);
    ct.out = (uint8_t* const*)(D + s.out);
    ct.cap = (const long long*)(D + s.cap);
    ct.bits = (unsigned long long*)(D + s.bits);
    ct.in_cnt = (const long long*)(D + s.in_cnt);
    ct.in_a = (const int*)(D + s.in_a);
    ct.out_cnt = (long long*)(D + s.out_cnt);
    ct.out_map = (AMap*)(D + s.out_map);
    ct.out_a = (int*)(D + s.out_a);
    ct.mode = mode;
    ct.chain_mode = nullptr;
    ct.modes_present = 1 << mode;
    ct.plane_segw = segw;
    ct.dct_bpl = dct_bpl;
    size_t o = 0;
    ct.flags = (int*)(E + o) + t0 * 4;
    o += cap_t * 16;
    ct.cnt = (long long*)(E + o) + t0 * 2 * kMaxCtx;
    o += cap_t * 16 * kMaxCtx;
    ct.maps = (AMap*)(E + o) + t0 * kMaxCtx;
    o += cap_t * sizeof(AMap) * kMaxCtx;
    ct.states = (int*)(E + o) + t0 * kMaxCtx;
    o += cap_t * 4 * kMaxCtx;
    ct.bitv = (unsigned long long*)(E + o) + t0 * 2;
    o += cap_t * 16;
    ct.edge = (uint32_t*)(E + o) + t0 * 2;
    ct.ticket = ticket;
    ct.ntiles = ntiles();
    ct.epoch = epoch;
    ct.nseg = (int)seg_r0.size();
    ct.seg_r0 = (const long long*)(D + s.seg_r0);
    ct.seg_t0 = (const long long*)(D + s.seg_t0);
    ct.seg_active = (const int*)(D + s.seg_active);
    ct.rr_chain = (const int*)(D + s.rr_chain);
    return ct;
  }
};

struct StagedParams {
  size_t qt, taps, pre, post;
};

// host staging bytes of one image's parameter blocks
inline size_t params_stage_bytes(const hdll_b200_image& im) {
  return 4 * kAlign + 256 * 8 + 8 * (2 * (size_t)std::max(0, im.params.radius) + 1) + im.hdr_pre_len + im.hdr_post_len;
}

template <class F>
inline StagedParams stage_params(F& stage, const hdll_b200_image& im) {
  const auto& p = im.params;
  StagedParams sp;
  double qt[256];  // luma, chroma, then their reciprocals (for the certified quantiser)
  quant_tables(p.quality, qt);
  for (int k = 0; k < 128; k++) qt[128 + k] = 1.0 / qt[k];
  sp.qt = stage(qt, sizeof(qt));
  sp.taps = stage(p.taps, (p.slrme && p.sigma_milli) ? 8 * (2 * (size_t)p.radius + 1) : 0);
  sp.pre = stage(im.hdr_pre, im.hdr_pre_len);
  sp.post = stage(im.hdr_post, im.hdr_post_len);
  return sp;
}

// Everything of an image's descriptor but the output fields.  mode: 0 full
// encode, 1 lossless plane (rgbe is the plane), 2 lossy image (rgbe is RGB).
inline void fill_desc(ImgDesc& d, const hdll_b200_image& im, const ImgLayout& L, uint8_t* B, int mode, bool any_trace,
                      const uint8_t* D, const StagedParams& sp) {
  const auto& p = im.params;
  memset(&d, 0, sizeof(d));
  d.w = im.width;
  d.h = im.height;
  d.n = (long long)d.w * d.h;
  d.pw = (d.w + 7) / 8 * 8;
  d.ph = (d.h + 7) / 8 * 8;
  d.nbx = d.pw / 8;
  d.nby = d.ph / 8;
  d.nblocks = (long long)d.nbx * d.nby;
  d.quality = p.quality;
  d.sigma_milli = p.sigma_milli;
  d.slrme = mode == 0 ? p.slrme : 0;
  d.global_regression = p.global_regression;
  d.blas_kernel = p.blas_kernel;
  d.blas_threads = p.blas_threads;
  d.radius = p.radius;
  d.want_trace = (any_trace && p.want_trace) ? 1 : 0;
  d.key = p.tmo_key;
  d.white_point = p.tmo_white_point;
  d.inv_gamma = p.tmo_inv_gamma;
  d.epsilon = p.tmo_epsilon;
  d.qt = (const double*)(D + sp.qt);
  d.taps = (const double*)(D + sp.taps);
  d.hdr_pre = D + sp.pre;
  d.hdr_pre_len = im.hdr_pre_len;
  d.hdr_post = D + sp.post;
  d.hdr_post_len = im.hdr_post_len;
  d.rgbe = mode == 2 ? nullptr : im.rgbe;
  d.sdr_in = mode == 2 ? im.rgbe : nullptr;
  d.crc_mask = mode == 0 ? 0x1F : (mode == 1 ? 0x2 : 0x1);
  d.maxlw = (unsigned long long*)(B + L.off_zero);
  d.status = (unsigned*)(B + L.off_zero + 8);
  d.amb = (unsigned*)(B + L.off_zero + 12);
  d.amb_list = (unsigned*)(B + L.off_amb);
  d.amb_cap = (unsigned)amb_cap(d.n);
  d.bin_count = (unsigned*)(B + L.off_zero + 16);
  d.sum_y = (long long*)(B + L.off_zero + 16 + 1024);
  d.isum = (long long*)(B + L.off_zero + 16 + 1024 + 8 * 768);
  d.int_fit = (mode == 0 && p.slrme && p.sigma_milli == 0) ? 1 : 0;
  d.full_n = d.n;
  d.pix_base = 0;
  d.node0 = 0;
  d.node1 = 1LL << pairwise_level(d.n);
  d.fit_p0 = 0;
  d.fit_m = d.n;
  d.fit_owner = 0;
  d.hist_fused = (d.slrme && !d.global_regression && mode == 0) ? 1 : 0;  // band.cu clears it
  d.crc_p0 = 0;
  d.crc_np = d.n;
  d.tm_nodes = (double*)(B + L.off_tmnodes);
  d.tm_level = pairwise_level(d.n);
  d.scalars = (double*)(B + L.off_scalars);
  d.sdr = d.want_trace ? B + L.off_sdr : nullptr;
  d.ycc = B + L.off_ycc;
  d.s_planes = B + L.off_s;
  d.zz = (int16_t*)(B + L.off_zz);
  d.sstar = L.off_sstar ? (double*)(B + L.off_sstar) : nullptr;
  d.sstar_tmp = L.off_sstar_tmp ? (double*)(B + L.off_sstar_tmp) : nullptr;
  d.e_plane = mode == 1 ? const_cast<uint8_t*>(im.rgbe) : B + L.off_e;
  d.res_planes = B + L.off_res;
  d.mstar = d.want_trace ? B + L.off_mstar : nullptr;
  d.sort_tiles = (int)((d.n + kSortTile - 1) / kSortTile);
  d.tile_hist = (unsigned*)(B + L.off_tile_hist);
  d.xs = (double*)(B + L.off_xs);
  d.ys = B + L.off_ys;
  d.bin_start = (unsigned*)(B + L.off_bin_start);
  d.seg_nodes = (double*)(B + L.off_seg_nodes);
  d.seg_level = (int*)(B + L.off_seg_level);
  d.seg_node_off = (long long*)(B + L.off_seg_node_off);
  d.dot_part = (double*)(B + L.off_dot);
  d.a32 = (float*)(B + L.off_a32);
  d.b32 = (float*)(B + L.off_b32);
  d.crc = (unsigned*)(B + L.off_crc);
  d.crc_part = (unsigned*)(B + L.off_crc_part);
  long long po = 0;
  for (int j = 0; j < 5; j++) {
    long long len = j == 0 ? 3 * d.n : d.n, csz = j == 0 ? kCrcChunkRgb : kCrcChunk;
    d.crc_chunks[j] = (len + csz - 1) / csz;
    d.crc_part_off[j] = po;
    po += d.crc_chunks[j];
  }
}

// entropy status arena of at least `ntiles` tiles, and a fresh launch epoch
inline int prepare_estat(Ctx* c, long long ntiles, cudaStream_t st) {
  if (ntiles > c->estat_tiles) {
    if (c->estat) cudaFree(c->estat);
    long long cap = ntiles + ntiles / 4 + 1024;
    size_t bytes = (size_t)cap * kEstatPerTile;
    CK(cudaMalloc(&c->estat, bytes));
    CK(cudaMemsetAsync(c->estat, 0, bytes, st));
    c->estat_tiles = cap;
    c->epoch = 0;
  }
  c->epoch++;
  if (c->epoch >= (1 << 28)) {  // epoch wrap: re-zero
    size_t bytes = (size_t)c->estat_tiles * kEstatPerTile;
    CK(cudaMemsetAsync(c->estat, 0, bytes, st));
    c->epoch = 1;
  }
  return HDLL_B200_OK;
}

void band_free(Ctx* c);  // band.cu

}  // namespace hdll_host
