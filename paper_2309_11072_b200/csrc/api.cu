// api.cu -- C ABI (include/hdll_b200.h) and batch orchestration.
//
// encode() order of stages (container.py:163-222), one launch per stage for
// the whole batch:
//   tonemap stats (tonemap.cu) -> base layer (base.cu) -> prefilter (prefilter.cu)
//   -> fit (fit.cu) -> estimate + residuals (estimate.cu) -> CRC-32 (crc.cu)
//   -> entropy coders, DCT + 4 planes (entropy.cu) -> serialize (assemble.cu)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>

#include "../../include/hdll_b200.h"
#include "encoder.cuh"

using namespace hdll;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// quantization_tables (codec_core.py:375-388)
void quant_tables(int quality, double* out128) {
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

inline long long dct_chain_cap(long long nblocks) { return (3 * nblocks * 544 + 64 + 15) / 16 * 16; }
inline long long plane_chain_cap(long long n) { return (n * 8 + 64 + 15) / 16 * 16; }
inline long long max_seg_nodes(long long n) { return 3 * (2 * (n / kNodeTarget) + 2 * 256 + 2); }

struct ImgLayout {
  size_t off_qt, off_taps, off_pre, off_post;
  size_t off_logv, off_tmnodes, off_scalars;
  size_t off_sdr, off_s, off_zz;
  size_t off_sstar, off_sstar_tmp, off_e, off_res, off_mstar;
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

constexpr size_t kZeroBytes = 8 /*maxlw*/ + 8 /*status, amb*/ + 1024 /*bin_count*/ + 8 * 768 /*sum_y*/;

struct Ctx {
  int device = 0;
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
  ImgDesc* d_descs = nullptr;
  // scratch for the host convenience path
  void* h2d = nullptr;
  size_t h2d_cap = 0;
  uint8_t* d_out = nullptr;
  size_t d_out_cap = 0;
  uint64_t* d_len = nullptr;
};

int cuda_fail(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fprintf(stderr, "hdll_b200: %s: %s\n", what, cudaGetErrorString(e));
    return HDLL_B200_E_CUDA;
  }
  return HDLL_B200_OK;
}
#define CK(x)                                      \
  do {                                             \
    int _rc = cuda_fail((x), #x);                  \
    if (_rc) return _rc;                           \
  } while (0)

int ensure(void** p, size_t* cap, size_t need, bool device, bool zero = false) {
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

ImgLayout plan(const hdll_b200_image& im, bool trace) {
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
  L.off_logv = take(sizeof(double) * n);
  L.off_tmnodes = take(sizeof(double) * ((size_t)1 << pairwise_level(n)));
  L.off_scalars = take(sizeof(double) * 4);
  L.off_sdr = trace ? take(3 * n) : 0;
  L.off_s = take(3 * n + 16);
  L.off_zz = take(sizeof(int16_t) * 3 * nb * 64);
  const bool real = im.params.slrme && im.params.sigma_milli != 0;
  L.off_sstar = real ? take(sizeof(double) * 3 * n) : 0;
  L.off_sstar_tmp = real ? take(sizeof(double) * 3 * n) : 0;
  L.off_e = take(n + 16);
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
  L.off_crc_part = take(sizeof(unsigned) * ((3 * n + 1019) / 1020 + 4 * ((n + kCrcChunk - 1) / kCrcChunk) + 8));
  L.chain_cap[0] = dct_chain_cap(nb);
  for (int k = 1; k < 5; k++) L.chain_cap[k] = plane_chain_cap(n);
  for (int k = 0; k < 5; k++) L.off_chain[k] = take(L.chain_cap[k]);
  L.total = o;
  return L;
}

int map_status(unsigned bits) {
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

  // chain of image i, kind k over `units` blocks / rows from `first`, DCT component cp (-1: all three)
  void add(int i, int k, int cp, long long fst, long long nunits, uint8_t* o, long long c) {
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
    const long long tiles = k == 0 ? (cp < 0 ? 3 : 1) * ((nunits + 31) / 32) : nunits;
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
    if (img.empty()) add(0, 1, -1, 0, 0, nullptr, 0);  // keep device arrays non-empty
  }
  size_t staged_bytes() const {
    size_t nc = img.size() + 2;
    return 16 * kAlign + 8 * (nc + 1) + 4 * nc * 3 + 8 * nc * 5 + (8 + 4 + 8 + sizeof(AMap)) * kMaxCtx * nc +
           8 * 2 * seg_r0.size() + 4 * seg_active.size() + 4 * rr_chain.size();
  }
  struct Staged {
    size_t tile_base, img, kind, comp, first, units, out, cap, bits, in_cnt, in_a, out_cnt, out_map, seg_r0, seg_t0,
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
    ct.mode = mode;
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

// mode: 0 full encode, 1 lossless plane (rgbe -> plane bytes), 2 lossy image (rgbe -> sdr rgb)
int run_batch(Ctx* c, const hdll_b200_image* imgs, int n, uint8_t* const* d_out, const uint64_t* out_cap,
              uint64_t* d_out_len, cudaStream_t st, int mode) {
  if (n <= 0) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  c->launches = 0;
  const bool any_trace = mode == 0;
  std::vector<ImgLayout> lays(n);
  size_t total = 0;
  std::vector<size_t> base(n);
  for (int i = 0; i < n; i++) {
    const auto& im = imgs[i];
    if (im.width == 0 || im.height == 0) return HDLL_B200_E_EMPTY;
    const auto& p = im.params;
    if (p.quality < 1 || p.quality > 100 || p.sigma_milli < 0 || p.sigma_milli > 65535 || p.blas_threads < 1 ||
        p.blas_kernel < 0 || p.blas_kernel > 1 || p.radius < 0)
      return HDLL_B200_E_ARG;
    if (p.slrme && p.sigma_milli && (!p.taps || p.radius < 1)) return HDLL_B200_E_ARG;
    if (((uintptr_t)im.rgbe & 15) != 0) return HDLL_B200_E_ARG;
    lays[i] = plan(im, any_trace && p.want_trace);
    base[i] = total;
    total += lays[i].total;
  }
  if (ensure(&c->arena, &c->arena_cap, total, true)) return HDLL_B200_E_CUDA;
  uint8_t* A = (uint8_t*)c->arena;

  // --- build descriptors and the host staging block (qt, taps, header bytes) ---
  std::vector<ImgDesc> ds(n);
  size_t stage_bytes = (size_t)n * 4 * kAlign;  // per-image alignment padding of the 4 staged blocks
  for (int i = 0; i < n; i++)
    stage_bytes += 256 * 8 + 8 * (2 * (size_t)std::max(0, imgs[i].params.radius) + 1) + imgs[i].hdr_pre_len +
                   imgs[i].hdr_post_len;
  // sequential-coder chains: the DCT stream of every image (kind 0) and its 4
  // plane streams (kinds 1..4), each family driven by its own kernel
  HostChains hc_dct, hc_pln;
  for (int i = 0; i < n; i++) {
    const long long w = imgs[i].width, h = imgs[i].height;
    const long long nb = ((w + 7) / 8) * ((h + 7) / 8);
    for (int k = 0; k < 5; k++) {
      bool active = (mode == 0) || (mode == 1 && k == 1) || (mode == 2 && k == 0);
      (k == 0 ? hc_dct : hc_pln).add(i, k, -1, 0, active ? (k == 0 ? nb : h) : 0, A + base[i] + lays[i].off_chain[k],
                                     lays[i].chain_cap[k]);
    }
  }
  hc_dct.schedule();
  hc_pln.schedule();
  const long long ntiles = hc_dct.ntiles() + hc_pln.ntiles();
  size_t tab_bytes = align_up(sizeof(ImgDesc) * n) + hc_dct.staged_bytes() + hc_pln.staged_bytes() + 16 * kAlign;
  // the batch that last used this staging slot may still read it
  const int slot = c->slot;
  c->slot ^= 1;
  if (c->slot_ev[slot]) CK(cudaEventSynchronize(c->slot_ev[slot]));
  else CK(cudaEventCreateWithFlags(&c->slot_ev[slot], cudaEventDisableTiming));
  if (ensure(&c->pinned_slot[slot], &c->pinned_cap_slot[slot], stage_bytes + tab_bytes + 4096, false))
    return HDLL_B200_E_CUDA;
  if (ensure(&c->tabs_slot[slot], &c->tabs_cap_slot[slot], stage_bytes + tab_bytes + 4096, true))
    return HDLL_B200_E_CUDA;
  c->tabs = c->tabs_slot[slot];
  uint8_t* H = (uint8_t*)c->pinned_slot[slot];
  uint8_t* D = (uint8_t*)c->tabs_slot[slot];
  size_t so = 0;
  auto stage = [&](const void* src, size_t bytes) {
    size_t r = so;
    if (bytes && src) memcpy(H + so, src, bytes);
    so = align_up(so + bytes);
    return r;
  };
  const size_t t_descs = stage(nullptr, sizeof(ImgDesc) * n);
  const HostChains::Staged sc_dct = hc_dct.stage(stage), sc_pln = hc_pln.stage(stage);
  const size_t t_ticket = stage(nullptr, 16);

  long long max_n = 0, max_sort_tiles = 0, max_nodes = 0, max_out = 0;
  int max_w = 0, max_h = 0, max_radius = 0, max_level = 0, max_base_tiles = 0, max_chunks = 1;
  bool any_real = false, any_slrme = false;
  for (int i = 0; i < n; i++) {
    const auto& im = imgs[i];
    const auto& p = im.params;
    const ImgLayout& L = lays[i];
    uint8_t* B = A + base[i];
    ImgDesc& d = ds[i];
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
    double qt[256];  // luma, chroma, then their reciprocals (for the certified quantiser)
    quant_tables(p.quality, qt);
    for (int k = 0; k < 128; k++) qt[128 + k] = 1.0 / qt[k];
    size_t s_qt = stage(qt, sizeof(qt));
    size_t s_taps = stage(p.taps, (p.slrme && p.sigma_milli) ? 8 * (2 * (size_t)p.radius + 1) : 0);
    size_t s_pre = stage(im.hdr_pre, im.hdr_pre_len);
    size_t s_post = stage(im.hdr_post, im.hdr_post_len);
    d.qt = (const double*)(D + s_qt);
    d.taps = (const double*)(D + s_taps);
    d.hdr_pre = D + s_pre;
    d.hdr_pre_len = im.hdr_pre_len;
    d.hdr_post = D + s_post;
    d.hdr_post_len = im.hdr_post_len;
    d.rgbe = mode == 2 ? nullptr : im.rgbe;
    d.sdr_in = mode == 2 ? im.rgbe : nullptr;
    d.crc_mask = mode == 0 ? 0x1F : (mode == 1 ? 0x2 : 0x1);
    d.maxlw = (unsigned long long*)(B + L.off_zero);
    d.status = (unsigned*)(B + L.off_zero + 8);
    d.amb = (unsigned*)(B + L.off_zero + 12);
    d.bin_count = (unsigned*)(B + L.off_zero + 16);
    d.sum_y = (long long*)(B + L.off_zero + 16 + 1024);
    d.full_n = d.n;
    d.pix_base = 0;
    d.px0 = 0;
    d.px1 = d.n;
    d.node0 = 0;
    d.node1 = 1LL << pairwise_level(d.n);
    d.fit_p0 = 0;
    d.fit_m = d.n;
    d.fit_owner = 0;
    d.crc_p0 = 0;
    d.crc_np = d.n;
    d.logv = (double*)(B + L.off_logv);
    d.tm_nodes = (double*)(B + L.off_tmnodes);
    d.tm_level = pairwise_level(d.n);
    d.scalars = (double*)(B + L.off_scalars);
    d.sdr = d.want_trace ? B + L.off_sdr : nullptr;
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
      long long len = j == 0 ? 3 * d.n : d.n, csz = j == 0 ? 1020 : kCrcChunk;
      d.crc_chunks[j] = (len + csz - 1) / csz;
      d.crc_part_off[j] = po;
      po += d.crc_chunks[j];
    }
    d.n_dct_tiles = (int)(3 * ((d.nblocks + 31) / 32));
    d.n_plane_tiles = 4 * d.h;
    d.out = mode == 0 ? d_out[i] : nullptr;
    d.out_len = mode == 0 ? (unsigned long long*)&d_out_len[i] : nullptr;
    d.out_cap = mode == 0 ? (long long)out_cap[i] : 0;
    max_n = std::max(max_n, d.n);
    max_w = std::max(max_w, d.w);
    max_h = std::max(max_h, d.h);
    max_radius = std::max(max_radius, d.radius);
    max_level = std::max(max_level, d.tm_level);
    max_sort_tiles = std::max(max_sort_tiles, (long long)d.sort_tiles);
    max_nodes = std::max(max_nodes, max_seg_nodes(d.n));
    max_chunks = std::max(max_chunks, std::min(d.blas_threads, kMaxBlasThreads));
    int tiles_x = (d.nbx + 15) / 16;
    max_base_tiles = std::max(max_base_tiles, tiles_x * d.nby);
    if (mode == 0) max_out = std::max(max_out, d.out_cap);
    any_real |= (d.slrme && d.sigma_milli != 0);
    any_slrme |= d.slrme != 0;
  }
  memcpy(H + t_descs, ds.data(), sizeof(ImgDesc) * n);
  memset(H + t_ticket, 0, 16);
  CK(cudaMemcpyAsync(D, H, so, cudaMemcpyHostToDevice, st));
  for (int i = 0; i < n; i++) CK(cudaMemsetAsync(A + base[i] + lays[i].off_zero, 0, kZeroBytes, st));
  c->d_descs = (ImgDesc*)(D + t_descs);
  const ImgDesc* dd = c->d_descs;

  // entropy status arena
  if (ntiles > c->estat_tiles) {
    if (c->estat) cudaFree(c->estat);
    long long cap = ntiles + ntiles / 4 + 1024;
    size_t bytes = (size_t)cap * kEstatPerTile;
    CK(cudaMalloc(&c->estat, bytes));
    CK(cudaMemset(c->estat, 0, bytes));
    c->estat_tiles = cap;
    c->epoch = 0;
  }
  c->epoch++;
  if (c->epoch >= (1 << 28)) {  // epoch wrap: re-zero
    size_t bytes = (size_t)c->estat_tiles * kEstatPerTile;
    CK(cudaMemsetAsync(c->estat, 0, bytes, st));
    c->epoch = 1;
  }
  uint8_t* E = (uint8_t*)c->estat;
  const long long cap_t = c->estat_tiles;
  ChainTab ct_dct = hc_dct.table(sc_dct, D, E, cap_t, 0, (int*)(D + t_ticket), c->epoch);
  ChainTab ct_pln = hc_pln.table(sc_pln, D, E, cap_t, hc_dct.ntiles(), (int*)(D + t_ticket) + 2, c->epoch);

  // --- stages ---
  if (!c->stage_ev[0])
    for (int k = 0; k <= kStages; k++) CK(cudaEventCreate(&c->stage_ev[k]));
  for (int k = 0; k < kStages; k++) c->stage_valid[k] = false;
  auto mark = [&](int k) {  // event k+1 closes stage k
    cudaEventRecord(c->stage_ev[k + 1], st);
    c->stage_valid[k] = true;
  };
  cudaEventRecord(c->stage_ev[0], st);
  if (mode == 0) {
    launch_tonemap_stats(dd, n, max_n, max_level, st);
    c->launches += 3;
  }
  mark(kStTonemap);
  if (mode != 1) {
    launch_base_layer(dd, n, max_base_tiles, st);
    c->launches += 1;
  }
  mark(kStBase);
  if (mode == 0 && any_real) {
    launch_prefilter(dd, n, max_w, max_h, max_radius, st);
    c->launches += 2;
  }
  mark(kStPrefilter);
  if (mode == 0 && any_slrme) {
    launch_fit(dd, n, (int)max_sort_tiles, max_nodes, max_chunks, st);
    c->launches += 7;
  }
  mark(kStFit);
  if (mode == 0) {
    launch_estimate(dd, n, max_n, st);
    c->launches += 1;
  }
  mark(kStEstimate);
  launch_crc(dd, n, max_n, st);
  c->launches += 2;
  mark(kStCrc);
  if (ct_dct.ntiles > 0) {
    launch_entropy_dct(dd, ct_dct, st);
    launch_entropy_fixup(ct_dct, st);
    c->launches += 2;
  }
  mark(kStEntropyDct);
  if (ct_pln.ntiles > 0) {
    launch_entropy_plane(dd, ct_pln, max_w, st);
    launch_entropy_fixup(ct_pln, st);
    c->launches += 2;
  }
  mark(kStEntropyPlane);
  if (mode == 0) {
    AsmTab at;
    at.dct_out = ct_dct.out;
    at.dct_bits = ct_dct.bits;
    at.plane_out = ct_pln.out;
    at.plane_bits = ct_pln.bits;
    launch_assemble(dd, n, at, max_out, st);
    c->launches += 1;
  }
  mark(kStAssemble);
  CK(cudaGetLastError());
  if (!c->done_ev) CK(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(c->done_ev, st));
  CK(cudaEventRecord(c->slot_ev[slot], st));
  c->last_stream = st;
  c->descs = ds;
  c->lays = lays;
  c->bits_off_dct = sc_dct.bits;
  c->bits_off_pln = sc_pln.bits;
  return HDLL_B200_OK;
}

int check_status(Ctx* c) {
  CK(cudaEventSynchronize(c->done_ev));
  unsigned worst = 0;
  for (auto& d : c->descs) {
    unsigned s = 0;
    CK(cudaMemcpy(&s, d.status, sizeof(s), cudaMemcpyDeviceToHost));
    worst |= s;
  }
  return map_status(worst);
}

}  // namespace

extern "C" {

int hdll_b200_ctx_create(hdll_b200_ctx** out, int device) {
  if (!out) return HDLL_B200_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return HDLL_B200_E_CUDA;
  CK(cudaSetDevice(device));
  Ctx* c = new Ctx();
  c->device = device;
  upload_base_constants();
  upload_crc_constants();
  CK(cudaGetLastError());
  *out = reinterpret_cast<hdll_b200_ctx*>(c);
  return HDLL_B200_OK;
}

void hdll_b200_ctx_destroy(hdll_b200_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->last_stream) cudaStreamSynchronize(c->last_stream);
  if (c->arena) cudaFree(c->arena);
  if (c->estat) cudaFree(c->estat);
  for (int k = 0; k < 2; k++) {
    if (c->tabs_slot[k]) cudaFree(c->tabs_slot[k]);
    if (c->pinned_slot[k]) cudaFreeHost(c->pinned_slot[k]);
    if (c->slot_ev[k]) cudaEventDestroy(c->slot_ev[k]);
  }
  if (c->h2d) cudaFreeHost(c->h2d);
  if (c->d_out) cudaFree(c->d_out);
  if (c->d_len) cudaFree(c->d_len);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  for (int k = 0; k <= kStages; k++)
    if (c->stage_ev[k]) cudaEventDestroy(c->stage_ev[k]);
  delete c;
}

uint64_t hdll_b200_stream_capacity(uint32_t w, uint32_t h, uint32_t pre, uint32_t post) {
  long long n = (long long)w * h;
  long long nb = (long long)((w + 7) / 8) * ((h + 7) / 8);
  return (uint64_t)(pre + 2 + 14 * 768 + post + 5 * 17 + dct_chain_cap(nb) + 4 * plane_chain_cap(n) + 64);
}

int hdll_b200_encode_batch_device(hdll_b200_ctx* ctx, const hdll_b200_image* imgs, int n, uint8_t* const* d_out,
                                  const uint64_t* out_cap, uint64_t* d_out_len, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !imgs || !d_out || !out_cap || !d_out_len) return HDLL_B200_E_ARG;
  for (int i = 0; i < n; i++)
    if (out_cap[i] < hdll_b200_stream_capacity(imgs[i].width, imgs[i].height, imgs[i].hdr_pre_len, imgs[i].hdr_post_len))
      return HDLL_B200_E_CAPACITY;
  int rc = run_batch(c, imgs, n, d_out, out_cap, d_out_len, (cudaStream_t)stream, 0);
  c->last_status = rc;
  return rc;
}

int hdll_b200_sync(hdll_b200_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return HDLL_B200_E_ARG;
  if (c->last_status) return c->last_status;
  if (!c->done_ev) return HDLL_B200_OK;
  return check_status(c);
}

int hdll_b200_encode_host(hdll_b200_ctx* ctx, const hdll_b200_image* img, uint8_t* h_out, uint64_t cap,
                          uint64_t* out_len) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !img || !h_out || !out_len) return HDLL_B200_E_ARG;
  if (img->width == 0 || img->height == 0) return HDLL_B200_E_EMPTY;
  CK(cudaSetDevice(c->device));
  const size_t in_bytes = (size_t)img->width * img->height * 4;
  const uint64_t ocap = hdll_b200_stream_capacity(img->width, img->height, img->hdr_pre_len, img->hdr_post_len);
  size_t dummy = c->d_out_cap;
  if (ensure((void**)&c->d_out, &dummy, align_up(in_bytes) + ocap, true)) return HDLL_B200_E_CUDA;
  c->d_out_cap = dummy;
  if (!c->d_len) CK(cudaMalloc(&c->d_len, 64));
  uint8_t* d_in = c->d_out;
  uint8_t* d_stream = c->d_out + align_up(in_bytes);
  CK(cudaMemcpy(d_in, img->rgbe, in_bytes, cudaMemcpyHostToDevice));
  hdll_b200_image im = *img;
  im.rgbe = d_in;
  uint8_t* outs[1] = {d_stream};
  uint64_t caps[1] = {ocap};
  int rc = run_batch(c, &im, 1, outs, caps, c->d_len, (cudaStream_t)0, 0);
  if (rc) return rc;
  rc = check_status(c);
  if (rc) return rc;
  uint64_t len = 0;
  CK(cudaMemcpy(&len, c->d_len, 8, cudaMemcpyDeviceToHost));
  *out_len = len;
  if (len > cap) return HDLL_B200_E_CAPACITY;
  CK(cudaMemcpy(h_out, d_stream, len, cudaMemcpyDeviceToHost));
  return HDLL_B200_OK;
}

int hdll_b200_trace(hdll_b200_ctx* ctx, int index, int which, uint8_t* h_dst, uint64_t nbytes) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || index < 0 || index >= (int)c->descs.size() || !h_dst) return HDLL_B200_E_ARG;
  const ImgDesc& d = c->descs[index];
  CK(cudaEventSynchronize(c->done_ev));
  const uint64_t n3 = 3 * (uint64_t)d.n;
  if (nbytes != n3) return HDLL_B200_E_ARG;
  if (which == 0 || which == 2) {
    const uint8_t* src = which == 0 ? d.sdr : d.mstar;
    if (!src) return HDLL_B200_E_ARG;
    CK(cudaMemcpy(h_dst, src, n3, cudaMemcpyDeviceToHost));
  } else if (which == 1) {  // decoded S as (h, w, 3)
    std::vector<uint8_t> planes(n3);
    CK(cudaMemcpy(planes.data(), d.s_planes, n3, cudaMemcpyDeviceToHost));
    for (long long p = 0; p < d.n; p++)
      for (int k = 0; k < 3; k++) h_dst[p * 3 + k] = planes[k * d.n + p];
  } else if (which == 3) {
    CK(cudaMemcpy(h_dst, d.res_planes, n3, cudaMemcpyDeviceToHost));
  } else {
    return HDLL_B200_E_ARG;
  }
  return HDLL_B200_OK;
}

static int plugin_common(Ctx* c, const uint8_t* h_src, size_t src_bytes, uint32_t w, uint32_t h, int quality, int mode,
                         uint8_t* h_body, uint64_t cap, uint64_t* body_len, uint32_t* crc, uint8_t* h_decoded) {
  if (w == 0 || h == 0) return HDLL_B200_E_EMPTY;
  CK(cudaSetDevice(c->device));
  size_t dummy = c->d_out_cap;
  if (ensure((void**)&c->d_out, &dummy, align_up(src_bytes) + 64, true)) return HDLL_B200_E_CUDA;
  c->d_out_cap = dummy;
  CK(cudaMemcpy(c->d_out, h_src, src_bytes, cudaMemcpyHostToDevice));
  hdll_b200_image im;
  memset(&im, 0, sizeof(im));
  im.rgbe = c->d_out;
  im.width = w;
  im.height = h;
  im.params.quality = quality;
  im.params.blas_threads = 1;
  int rc = run_batch(c, &im, 1, nullptr, nullptr, nullptr, (cudaStream_t)0, mode);
  if (rc) return rc;
  rc = check_status(c);
  if (rc) return rc;
  const ImgDesc& d = c->descs[0];
  const int k = mode == 1 ? 1 : 0;
  const ImgLayout& L = c->lays[0];
  uint8_t* chain = (uint8_t*)c->arena + L.off_chain[k];
  unsigned long long bits = 0;
  // mode 1: the only plane chain is image 0's E chain (index 1 of 4); mode 2: the DCT chain
  const size_t boff = mode == 1 ? c->bits_off_pln + 8 * 0 : c->bits_off_dct;
  CK(cudaMemcpy(&bits, (uint8_t*)c->tabs + boff, 8, cudaMemcpyDeviceToHost));
  const uint64_t nbytes = (bits + 7) / 8;
  *body_len = 8 + nbytes;
  if (8 + nbytes > cap) return HDLL_B200_E_CAPACITY;
  uint32_t wh[2] = {w, h};
  memcpy(h_body, wh, 8);
  CK(cudaMemcpy(h_body + 8, chain, nbytes, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(crc, d.crc + (mode == 1 ? 1 : 0), 4, cudaMemcpyDeviceToHost));
  if (h_decoded) {
    std::vector<uint8_t> planes(3 * (size_t)d.n);
    CK(cudaMemcpy(planes.data(), d.s_planes, planes.size(), cudaMemcpyDeviceToHost));
    for (long long p = 0; p < d.n; p++)
      for (int q = 0; q < 3; q++) h_decoded[p * 3 + q] = planes[q * d.n + p];
  }
  return HDLL_B200_OK;
}

int hdll_b200_lossless_encode_plane(hdll_b200_ctx* ctx, const uint8_t* h_plane, uint32_t w, uint32_t h,
                                    uint8_t* h_body, uint64_t cap, uint64_t* body_len, uint32_t* crc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !h_plane || !h_body || !body_len || !crc) return HDLL_B200_E_ARG;
  return plugin_common(c, h_plane, (size_t)w * h, w, h, 85, 1, h_body, cap, body_len, crc, nullptr);
}

int hdll_b200_lossy_encode(hdll_b200_ctx* ctx, const uint8_t* h_rgb, uint32_t w, uint32_t h, int32_t quality,
                           uint8_t* h_body, uint64_t cap, uint64_t* body_len, uint8_t* h_decoded, uint32_t* crc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !h_rgb || !h_body || !body_len || !crc || !h_decoded) return HDLL_B200_E_ARG;
  if (quality < 1 || quality > 100) return HDLL_B200_E_ARG;
  return plugin_common(c, h_rgb, (size_t)w * h * 3, w, h, quality, 2, h_body, cap, body_len, crc, h_decoded);
}

int hdll_b200_last_launch_count(hdll_b200_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  return c ? c->launches : 0;
}

int hdll_b200_stage_times(hdll_b200_ctx* ctx, float* ms, int n) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !ms || n < kStages || !c->stage_ev[0]) return HDLL_B200_E_ARG;
  CK(cudaEventSynchronize(c->stage_ev[kStages]));
  for (int k = 0; k < kStages; k++) {
    ms[k] = 0.f;
    if (c->stage_valid[k]) CK(cudaEventElapsedTime(&ms[k], c->stage_ev[k], c->stage_ev[k + 1]));
  }
  return HDLL_B200_OK;
}

const char* hdll_b200_status_string(int s) {
  switch (s) {
    case HDLL_B200_OK: return "ok";
    case HDLL_B200_E_ARG: return "invalid argument";
    case HDLL_B200_E_EMPTY: return "cannot encode an empty image";
    case HDLL_B200_E_NONFINITE: return "regression parameters must be finite";
    case HDLL_B200_E_CUDA: return "CUDA error";
    case HDLL_B200_E_INTERNAL: return "internal device error";
    case HDLL_B200_E_CAPACITY: return "output capacity exceeded";
    default: return "unknown status";
  }
}

}  // extern "C"
