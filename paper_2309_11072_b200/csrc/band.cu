// band.cu -- row-band encoder for tile-sharded single images (SURVEY.md 8e,
// BASELINE config 3), C ABI in include/hdll_b200.h (hdll_b200_band_*).
//
// The reference encodes an image in one sequential pass (container.py:131-230).
// Split into contiguous row bands, one per rank, every stage is local to a
// band except four global dependencies, each crossed by one exchange of a
// small summary (the host does the exchange between the phases below):
//   1. tone-map log-average: numpy's pairwise tree (tonemap.py:101) is cut at
//      depth L; each rank sums its nodes, all ranks combine all 2^L nodes in
//      the same fixed tree (k_tm_scalars), so every rank gets the same bits;
//   2. SLRME fit (estimator.py:172-214): the sums are order dependent, so each
//      exponent bin is fitted by one owner rank from every band's samples of
//      that bin in band order, which is raster order (all-to-all exchange);
//   3. the adaptive Rice coders (_kernels.py:169-216, 280-324): a band's slice
//      of a stream is a chain piece; counts, then A-maps (common.cuh AMap),
//      then bit lengths are prefix-combined over the pieces in stream order;
//   4. CRC-32 (codec_core.py:252-253): zlib's crc32_combine of band CRCs.
// A band recomputes the halo rows it needs (one DCT block row above for the DC
// predictor and the prefilter / plane-coder neighbourhoods) from the RGBE
// rows it holds, so no pixel data crosses ranks except the fit samples.
#include <chrono>
#include <cstdlib>

#include "host_common.cuh"
#include "pairwise.cuh"

using namespace hdll;
using namespace hdll_host;

namespace hdll_host {

constexpr int kPieces = HDLL_B200_BAND_PIECES;

struct Band {
  int W = 0, H = 0, y0 = 0, y1 = 0, c0 = 0, c1 = 0;
  int level = 0;
  long long node0 = 0, node1 = 0;
  hdll_b200_image im{};  // the band image: rows [c0, c1)
  ImgLayout L{};
  ImgDesc desc{};
  cudaStream_t st = nullptr;
  std::vector<uint32_t> hist;
  // device memory
  void* arena = nullptr;  // band arrays (plan())
  size_t arena_cap = 0;
  void* tabs = nullptr;  // desc, parameters, nodes, chain tables
  size_t tabs_cap = 0;
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  void* pieces = nullptr;  // the 7 piece streams
  size_t pieces_cap = 0;
  void* own = nullptr;  // owner fit
  size_t own_cap = 0;
  void* asmb = nullptr;  // rank-0 assembly
  size_t asmb_cap = 0;
  ImgDesc* d_desc = nullptr;
  long long crc_units = 0;
  double* d_nodes = nullptr;
  uint8_t* piece_ptr[kPieces] = {};
  HostChains hc_dct, hc_pln;
  HostChains::Staged sc_dct{}, sc_pln{};
  int* d_ticket = nullptr;
  size_t t_cmode = 0;  // per-chain modes in tabs: DCT chains at +0, plane chains at +16
};

void band_free(Ctx* c) {
  Band* b = c->band;
  if (!b) return;
  for (void* p : {b->arena, b->tabs, b->pieces, b->own, b->asmb})
    if (p) cudaFree(p);
  if (b->pinned) cudaFreeHost(b->pinned);
  delete b;
  c->band = nullptr;
}

}  // namespace hdll_host

namespace {

// HDLL_B200_BAND_TIMING=1: host time of band_begin's steps on stderr (diagnostic)
struct StepClock {
  bool on = std::getenv("HDLL_B200_BAND_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "band_begin %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// pixel range of depth-L node idx of the pairwise tree over n (pairwise.cuh)
void node_range(long long n, int L, long long idx, long long* p0, long long* p1) {
  long long off, sz;
  pairwise_node(n, L, idx, &off, &sz);
  *p0 = off;
  *p1 = off + sz;
}

int sync_status(Band* b) {
  CK(cudaStreamSynchronize(b->st));
  CK(cudaGetLastError());
  return HDLL_B200_OK;
}

// run the 7 piece chains, piece k in modes[k] (entropy.cu ChainTab: 0 code,
// 1 counts, 2 A-maps, kModeSkip not run)
int run_chains(Ctx* c, Band* b, const int* modes) {
  int pres_dct = 0, pres_pln = 0;
  for (int k = 0; k < kPieces; k++)
    if (modes[k] != kModeSkip) (k < 3 ? pres_dct : pres_pln) |= 1 << modes[k];
  if (!pres_dct && !pres_pln) return HDLL_B200_OK;
  const long long ntiles = b->hc_dct.ntiles() + b->hc_pln.ntiles();
  if (int rc = prepare_estat(c, ntiles, b->st)) return rc;
  CK(cudaMemsetAsync(b->d_ticket, 0, 16, b->st));
  uint8_t* D = (uint8_t*)b->tabs;
  CK(cudaMemcpyAsync(D + b->t_cmode, modes, 4 * 3, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(D + b->t_cmode + 16, modes + 3, 4 * 4, cudaMemcpyHostToDevice, b->st));
  uint8_t* E = (uint8_t*)c->estat;
  ChainTab ct_dct = b->hc_dct.table(b->sc_dct, D, E, c->estat_tiles, 0, b->d_ticket, c->epoch, 0);
  ChainTab ct_pln = b->hc_pln.table(b->sc_pln, D, E, c->estat_tiles, b->hc_dct.ntiles(), b->d_ticket + 2, c->epoch, 0);
  ct_dct.chain_mode = (const int*)(D + b->t_cmode);
  ct_pln.chain_mode = (const int*)(D + b->t_cmode + 16);
  ct_dct.modes_present = pres_dct;
  ct_pln.modes_present = pres_pln;
  if (ensure(&c->plane_scratch, &c->plane_scratch_cap,
             std::max(dct_scratch_bytes(ct_dct), plane_scratch_bytes(ct_pln, b->W)), true))
    return HDLL_B200_E_CUDA;
  if (pres_dct) {
    launch_entropy_dct(b->d_desc, ct_dct, c->plane_scratch, b->st);
    launch_entropy_fixup(ct_dct, b->st);
    c->launches += 2;
  }
  if (pres_pln) {
    launch_entropy_plane(b->d_desc, ct_pln, b->W, c->plane_scratch, b->st);
    launch_entropy_fixup(ct_pln, b->st);
    c->launches += 2;
  }
  return sync_status(b);
}

// copy a per-chain [kMaxCtx] array between the host piece order (3 DCT, 4 planes) and the two chain tables
template <class T>
int pieces_to_dev(Band* b, size_t off_dct, size_t off_pln, const T* h) {
  uint8_t* D = (uint8_t*)b->tabs;
  CK(cudaMemcpyAsync(D + off_dct, h, sizeof(T) * 3 * kMaxCtx, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(D + off_pln, h + 3 * kMaxCtx, sizeof(T) * 4 * kMaxCtx, cudaMemcpyHostToDevice, b->st));
  return HDLL_B200_OK;
}
template <class T>
int pieces_from_dev(Band* b, size_t off_dct, size_t off_pln, T* h) {
  uint8_t* D = (uint8_t*)b->tabs;
  CK(cudaMemcpyAsync(h, D + off_dct, sizeof(T) * 3 * kMaxCtx, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h + 3 * kMaxCtx, D + off_pln, sizeof(T) * 4 * kMaxCtx, cudaMemcpyDeviceToHost, b->st));
  return sync_status(b);
}

inline size_t fit_chunk_bytes(long long m) { return 24 * (size_t)m + ((3 * (size_t)m + 7) & ~(size_t)7); }

Band* band_of(hdll_b200_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  return c ? c->band : nullptr;
}

}  // namespace

extern "C" {

int hdll_b200_band_begin(hdll_b200_ctx* ctx, const hdll_b200_image* img, const hdll_b200_band* band, void* stream,
                         double* h_nodes, double* h_maxlw) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  if (!c || !img || !band || !h_nodes || !h_maxlw) return HDLL_B200_E_ARG;
  if (img->width == 0 || img->height == 0) return HDLL_B200_E_EMPTY;
  const auto& p = img->params;
  if (p.quality < 1 || p.quality > 100 || p.sigma_milli < 0 || p.sigma_milli > 65535 || p.blas_threads < 1 ||
      p.blas_kernel < 0 || p.blas_kernel > 1 || p.radius < 0)
    return HDLL_B200_E_ARG;
  if (p.slrme && p.sigma_milli && (!p.taps || p.radius < 1)) return HDLL_B200_E_ARG;
  if (((uintptr_t)img->rgbe & 15) != 0) return HDLL_B200_E_ARG;
  const int W = (int)img->width, H = (int)img->height;
  const long long full_n = (long long)W * H;
  const int level = pairwise_level(full_n);
  const hdll_b200_band& bd = *band;
  if (!(bd.crow0 <= bd.row0 && bd.row0 < bd.row1 && bd.row1 <= bd.crow1 && bd.crow1 <= (uint32_t)H) ||
      bd.row0 % 8 || (bd.row1 % 8 && bd.row1 != (uint32_t)H) || bd.crow0 % 8 ||
      (bd.crow1 % 8 && bd.crow1 != (uint32_t)H) || bd.node0 > bd.node1 || bd.node1 > (1ULL << level))
    return HDLL_B200_E_ARG;
  // halo: the DCT block row above (DC predictor) and the prefilter / plane-coder rows
  const int rad = (p.slrme && p.sigma_milli) ? p.radius : 0;
  if (bd.row0 > 0 && ((int)bd.row0 - (int)bd.crow0 < std::max(8, rad + 1))) return HDLL_B200_E_ARG;
  if (bd.row1 < (uint32_t)H && (int)bd.crow1 - (int)bd.row1 < rad) return HDLL_B200_E_ARG;
  long long px0 = bd.row0 * (long long)W, px1 = px0;
  if (bd.node1 > bd.node0) {
    long long a, e;
    node_range(full_n, level, (long long)bd.node0, &px0, &e);
    node_range(full_n, level, (long long)bd.node1 - 1, &a, &px1);
  }
  if (px0 < (long long)bd.crow0 * W || px1 > (long long)bd.crow1 * W) return HDLL_B200_E_ARG;
  StepClock clk;
  CK(cudaSetDevice(c->device));
  if (clk.on) {
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    clk.mark("pending work on the stream");
  }
  if (c->done_ev) CK(cudaEventSynchronize(c->done_ev));  // the shared coder scratch of an encode batch
  clk.mark("sync");
  c->launches = 0;
  if (!c->band) c->band = new Band();
  Band* b = c->band;
  b->W = W;
  b->H = H;
  b->y0 = (int)bd.row0;
  b->y1 = (int)bd.row1;
  b->c0 = (int)bd.crow0;
  b->c1 = (int)bd.crow1;
  b->level = level;
  b->node0 = (long long)bd.node0;
  b->node1 = (long long)bd.node1;
  b->st = (cudaStream_t)stream;
  b->im = *img;
  b->im.height = (uint32_t)(b->c1 - b->c0);
  b->im.hdr_pre = nullptr;
  b->im.hdr_pre_len = 0;
  b->im.hdr_post = nullptr;
  b->im.hdr_post_len = 0;
  b->im.params.want_trace = 0;
  b->L = plan(b->im, false);
  if (ensure(&b->arena, &b->arena_cap, b->L.total, true)) return HDLL_B200_E_CUDA;
  uint8_t* B = (uint8_t*)b->arena;
  clk.mark("arena");

  // chain pieces: Y, Cb, Cr of the band's block rows, then the E, R, G, B rows
  const int nbx = (W + 7) / 8;
  const long long bfirst = (long long)(b->y0 - b->c0) / 8 * nbx;
  const long long bunits = (long long)((b->y1 + 7) / 8 - b->y0 / 8) * nbx;
  const long long rows = b->y1 - b->y0;
  const size_t dct_cap = (size_t)((bunits * 544 + 64 + 15) / 16 * 16);
  const size_t pln_cap = (size_t)plane_chain_cap(rows * W);
  if (ensure(&b->pieces, &b->pieces_cap, 3 * dct_cap + 4 * pln_cap + 1024, true)) return HDLL_B200_E_CUDA;
  {
    uint8_t* P = (uint8_t*)b->pieces;
    for (int k = 0; k < kPieces; k++) {
      b->piece_ptr[k] = P;
      P += k < 3 ? dct_cap : pln_cap;
    }
  }
  b->hc_dct = HostChains();
  b->hc_pln = HostChains();
  b->hc_dct.dct_bpl = kDctMaxBlocksPerLane;  // as the whole-image encode (api.cu)
  for (int cp = 0; cp < 3; cp++) b->hc_dct.add(0, 0, cp, bfirst, bunits, b->piece_ptr[cp], (long long)dct_cap, W);
  b->hc_pln.segw = plane_segw_for(4 * rows, W);
  for (int k = 1; k < 5; k++)
    b->hc_pln.add(0, k, -1, b->y0 - b->c0, rows, b->piece_ptr[2 + k], (long long)pln_cap, W);
  b->hc_dct.schedule();
  b->hc_pln.schedule();
  clk.mark("chains");

  // host staging -> tabs: desc, parameters, nodes (reserved), chain tables, tickets
  const size_t nodes_bytes = sizeof(double) * ((size_t)1 << level);
  const size_t tab_bytes = align_up(sizeof(ImgDesc)) + params_stage_bytes(b->im) + align_up(nodes_bytes) +
                           b->hc_dct.staged_bytes() + b->hc_pln.staged_bytes() + 8 * kAlign;
  if (ensure(&b->pinned, &b->pinned_cap, tab_bytes, false)) return HDLL_B200_E_CUDA;
  if (ensure(&b->tabs, &b->tabs_cap, tab_bytes, true)) return HDLL_B200_E_CUDA;
  uint8_t* Hs = (uint8_t*)b->pinned;
  uint8_t* D = (uint8_t*)b->tabs;
  size_t so = 0;
  auto stage = [&](const void* src, size_t bytes) {
    size_t r = so;
    if (bytes && src) memcpy(Hs + so, src, bytes);
    so = align_up(so + bytes);
    return r;
  };
  const size_t t_desc = stage(nullptr, sizeof(ImgDesc));
  const StagedParams sp = stage_params(stage, b->im);
  const size_t t_nodes = stage(nullptr, nodes_bytes);
  b->sc_dct = b->hc_dct.stage(stage);
  b->sc_pln = b->hc_pln.stage(stage);
  const size_t t_ticket = stage(nullptr, 16);
  b->t_cmode = stage(nullptr, 32);
  ImgDesc& d = b->desc;
  fill_desc(d, b->im, b->L, B, 0, false, D, sp);
  d.full_n = full_n;
  d.pix_base = (long long)b->c0 * W;
  d.node0 = b->node0;
  d.node1 = b->node1;
  d.tm_level = level;
  d.tm_nodes = (double*)(D + t_nodes);
  d.fit_p0 = (long long)(b->y0 - b->c0) * W;
  d.fit_m = rows * W;
  d.sort_tiles = (int)((d.fit_m + kSortTile - 1) / kSortTile);
  d.hist_fused = 0;  // the band's fit rows are a sub-range: k_sort_hist counts them
  // sigma > 0: bins are fitted by their owner rank from the exchanged samples;
  // sigma = 0 (int_fit from fill_desc): every rank sums its rows' exact
  // integer bins and the ranks all-reduce the table (hdll_b200_band_fit_sums)
  d.crc_p0 = d.fit_p0;
  d.crc_np = d.fit_m;
  b->crc_units = crc_assign_units(&d, 1);
  b->d_desc = (ImgDesc*)(D + t_desc);
  b->d_nodes = d.tm_nodes;
  b->d_ticket = (int*)(D + t_ticket);
  memcpy(Hs + t_desc, &d, sizeof(ImgDesc));
  clk.mark("staging");
  CK(cudaMemcpyAsync(D, Hs, so, cudaMemcpyHostToDevice, b->st));
  if (clk.on) {
    CK(cudaStreamSynchronize(b->st));
    clk.mark("upload");
  }
  CK(cudaMemsetAsync(B + b->L.off_zero, 0, kZeroBytes, b->st));
  if (clk.on) {
    CK(cudaStreamSynchronize(b->st));
    clk.mark("memset");
  }
  launch_tonemap_partial(b->d_desc, 1, d.n, level, b->st);
  if (clk.on) {
    CK(cudaStreamSynchronize(b->st));
    clk.mark("tonemap");
    fprintf(stderr, "band_begin staged %zu bytes, nodes [%lld, %lld) of 2^%d, n %lld\n", so, b->node0, b->node1, level, d.n);
  }
  c->launches += 2;
  const size_t nn = (size_t)(b->node1 - b->node0);
  if (nn) CK(cudaMemcpyAsync(h_nodes, b->d_nodes + b->node0, sizeof(double) * nn, cudaMemcpyDeviceToHost, b->st));
  unsigned long long mx = 0;
  CK(cudaMemcpyAsync(&mx, d.maxlw, 8, cudaMemcpyDeviceToHost, b->st));
  if (int rc = sync_status(b)) return rc;
  clk.mark("readback");
  memcpy(h_maxlw, &mx, 8);
  return HDLL_B200_OK;
}

int hdll_b200_band_layers(hdll_b200_ctx* ctx, const double* h_nodes_all, uint64_t n_nodes, double maxlw,
                          uint32_t* h_hist) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_nodes_all || !h_hist || n_nodes != (1ULL << b->level) || !(maxlw >= 0.0)) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  CK(cudaMemcpyAsync(b->d_nodes, h_nodes_all, sizeof(double) * n_nodes, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(d.maxlw, &maxlw, 8, cudaMemcpyHostToDevice, b->st));
  launch_tonemap_scalars(b->d_desc, 1, b->st);
  launch_base_layer(b->d_desc, 1, (d.nbx + 15) / 16 * d.nby, d.n, b->st);
  c->launches += 3;
  if (d.slrme && d.sigma_milli) {
    launch_prefilter(b->d_desc, 1, d.w, d.h, d.radius, b->st);
    c->launches += 2;
  }
  b->hist.assign(256, 0);
  if (d.slrme && d.int_fit) {  // sigma = 0: the band's exact bin sums, no sort
    launch_fit_hist(b->d_desc, 1, d.sort_tiles, b->st);
    launch_fit_int_sums(b->d_desc, 1, d.fit_m, b->st);
    c->launches += 2;
    CK(cudaMemcpyAsync(b->hist.data(), d.bin_count, 4 * 256, cudaMemcpyDeviceToHost, b->st));
  } else if (d.slrme) {
    launch_fit_sort(b->d_desc, 1, d.sort_tiles, b->st);
    c->launches += 3;
    CK(cudaMemcpyAsync(b->hist.data(), d.bin_count, 4 * 256, cudaMemcpyDeviceToHost, b->st));
  }
  if (int rc = sync_status(b)) return rc;
  memcpy(h_hist, b->hist.data(), 4 * 256);
  return HDLL_B200_OK;
}

int hdll_b200_band_fit_sums(hdll_b200_ctx* ctx, int64_t* h_sums) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_sums || !b->desc.int_fit) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  CK(cudaMemcpyAsync(h_sums, d.isum, 8 * 3 * 768, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h_sums + 3 * 768, d.sum_y, 8 * 768, cudaMemcpyDeviceToHost, b->st));
  return sync_status(b);
}

int hdll_b200_band_fit_coef(hdll_b200_ctx* ctx, const int64_t* h_sums, const uint32_t* h_hist, float* h_a32,
                            float* h_b32, uint32_t* h_status) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_sums || !h_hist || !h_a32 || !h_b32 || !h_status || !b->desc.int_fit) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  // the whole image's table replaces the band's: counts, sums of x, x^2, x*y and y
  CK(cudaMemcpyAsync(d.bin_count, h_hist, 4 * 256, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(d.isum, h_sums, 8 * 3 * 768, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(d.sum_y, h_sums + 3 * 768, 8 * 768, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemsetAsync(d.a32, 0, 4 * 768, b->st));
  CK(cudaMemsetAsync(d.b32, 0, 4 * 768, b->st));
  launch_fit_int_coef(b->d_desc, 1, b->st);
  c->launches += 1;
  CK(cudaMemcpyAsync(h_a32, d.a32, 4 * 768, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h_b32, d.b32, 4 * 768, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h_status, d.status, 4, cudaMemcpyDeviceToHost, b->st));
  return sync_status(b);
}

int hdll_b200_band_fit_local(hdll_b200_ctx* ctx, float* h_a32, float* h_b32, uint32_t* h_status) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_a32 || !h_b32 || !h_status || b->desc.int_fit) return HDLL_B200_E_ARG;
  if (b->y0 != 0 || b->y1 != b->H) return HDLL_B200_E_ARG;  // the band must be the whole image
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  CK(cudaMemsetAsync(d.a32, 0, 4 * 768, b->st));
  CK(cudaMemsetAsync(d.b32, 0, 4 * 768, b->st));
  if (d.slrme) {  // the band's samples, sorted by phase 2, are every sample of the image
    launch_fit_bins(b->d_desc, 1, max_seg_nodes(d.fit_m), std::min(d.blas_threads, kMaxBlasThreads), b->st);
    c->launches += 4;
  }
  CK(cudaMemcpyAsync(h_a32, d.a32, 4 * 768, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h_b32, d.b32, 4 * 768, cudaMemcpyDeviceToHost, b->st));
  CK(cudaMemcpyAsync(h_status, d.status, 4, cudaMemcpyDeviceToHost, b->st));
  return sync_status(b);
}

int hdll_b200_band_fit_send(hdll_b200_ctx* ctx, const uint32_t* owner_lo, int nowners, uint8_t* d_send,
                            uint64_t send_cap, uint64_t* h_send_bytes) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !owner_lo || nowners < 1 || !h_send_bytes || b->hist.size() != 256) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  const long long m = d.fit_m;
  std::vector<long long> bs(257, 0);
  for (int e = 0; e < 256; e++) bs[e + 1] = bs[e] + b->hist[e];
  uint64_t off = 0;
  for (int o = 0; o < nowners; o++) {
    long long s0 = 0, s1 = 0;
    if (d.slrme) {
      if (d.global_regression) {  // one raster-order segment, fitted by owner 0
        s0 = o == 0 ? 0 : m;
        s1 = m;
      } else {
        const uint32_t lo = owner_lo[o], hi = owner_lo[o + 1];
        if (lo > hi || hi > 256) return HDLL_B200_E_ARG;
        s0 = bs[lo];
        s1 = bs[hi];
      }
    }
    const long long mo = s1 - s0;
    const size_t bytes = fit_chunk_bytes(mo);
    if (off + bytes > send_cap) return HDLL_B200_E_CAPACITY;
    for (int ch = 0; ch < 3 && mo > 0; ch++) {
      CK(cudaMemcpyAsync(d_send + off + 8 * (size_t)ch * mo, d.xs + ch * m + s0, 8 * (size_t)mo,
                         cudaMemcpyDeviceToDevice, b->st));
      CK(cudaMemcpyAsync(d_send + off + 24 * (size_t)mo + (size_t)ch * mo, d.ys + ch * m + s0, (size_t)mo,
                         cudaMemcpyDeviceToDevice, b->st));
    }
    h_send_bytes[o] = bytes;
    off += bytes;
  }
  return sync_status(b);
}

int hdll_b200_band_fit_owner(hdll_b200_ctx* ctx, const uint8_t* d_recv, const uint64_t* h_recv_bytes,
                             const uint32_t* h_hist, int nsrc, uint32_t e_lo, uint32_t e_hi, float* h_a32,
                             float* h_b32, uint32_t* h_status) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_recv_bytes || !h_hist || nsrc < 1 || e_lo > e_hi || e_hi > 256 || !h_a32 || !h_b32 || !h_status)
    return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  memset(h_a32, 0, 4 * 768);
  memset(h_b32, 0, 4 * 768);
  *h_status = 0;
  const ImgDesc& bd = b->desc;
  if (!bd.slrme) return HDLL_B200_OK;
  const bool glob = bd.global_regression != 0;
  // per-source sample counts and bin offsets; destination offsets (bins, then sources)
  std::vector<long long> src_m(nsrc, 0), src_off(nsrc + 1, 0);
  std::vector<unsigned> src_bin(nsrc * 257, 0), dst_bin(nsrc * 256, 0), gcount(256, 0), gstart(257, 0);
  for (int s = 0; s < nsrc; s++) {
    const uint32_t* hs = h_hist + 256 * s;
    unsigned run = 0;
    for (int e = 0; e < 256; e++) {
      src_bin[s * 257 + e] = run;
      const unsigned cnt = !glob && (uint32_t)e >= e_lo && (uint32_t)e < e_hi ? hs[e] : 0u;
      run += cnt;
      gcount[e] += cnt;
    }
    if (glob && e_lo < e_hi) {  // a single raster-order segment in "bin" 0, all on this owner
      for (int e = 0; e < 256; e++) run += hs[e];
      for (int e = 1; e <= 256; e++) src_bin[s * 257 + e] = (unsigned)run;
      gcount[0] += (unsigned)run;
    }
    src_bin[s * 257 + 256] = run;
    src_m[s] = run;
    if (h_recv_bytes[s] != fit_chunk_bytes(run)) return HDLL_B200_E_ARG;
    src_off[s + 1] = src_off[s] + (long long)h_recv_bytes[s];
  }
  for (int e = 0; e < 256; e++) gstart[e + 1] = gstart[e] + gcount[e];
  const long long M = gstart[256];
  for (int e = 0; e < 256; e++) {
    unsigned run = gstart[e];
    for (int s = 0; s < nsrc; s++) {
      dst_bin[s * 256 + e] = run;
      run += src_bin[s * 257 + e + 1] - src_bin[s * 257 + e];
    }
  }
  // owner arena: desc, tables, samples, fit scratch
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  const size_t o_desc = take(sizeof(ImgDesc)), o_zero = take(kZeroBytes), o_start = take(4 * 257);
  const size_t o_srcoff = take(8 * (nsrc + 1)), o_srcm = take(8 * nsrc), o_srcbin = take(4 * 257 * (size_t)nsrc);
  const size_t o_dstbin = take(4 * 256 * (size_t)nsrc);
  const size_t o_xs = take(8 * 3 * (size_t)M + 16), o_ys = take(3 * (size_t)M + 16);
  const size_t o_nodes = take(sizeof(double) * max_seg_nodes(M)), o_level = take(4 * 768), o_noff = take(8 * 769);
  const size_t o_dot = take(sizeof(double) * 768 * kMaxBlasThreads * 2), o_a = take(4 * 768), o_b = take(4 * 768);
  if (ensure(&b->own, &b->own_cap, o, true)) return HDLL_B200_E_CUDA;
  uint8_t* O = (uint8_t*)b->own;
  ImgDesc d;
  memset(&d, 0, sizeof(d));
  d.slrme = 1;
  d.fit_owner = 1;
  d.global_regression = bd.global_regression;
  d.blas_kernel = bd.blas_kernel;
  d.blas_threads = bd.blas_threads;
  d.sigma_milli = bd.sigma_milli;
  d.n = M;
  d.fit_m = M;
  d.status = (unsigned*)(O + o_zero + 8);
  d.bin_count = (unsigned*)(O + o_zero + 16);
  d.sum_y = (long long*)(O + o_zero + 16 + 1024);
  d.bin_start = (unsigned*)(O + o_start);
  d.xs = (double*)(O + o_xs);
  d.ys = O + o_ys;
  d.seg_nodes = (double*)(O + o_nodes);
  d.seg_level = (int*)(O + o_level);
  d.seg_node_off = (long long*)(O + o_noff);
  d.dot_part = (double*)(O + o_dot);
  d.a32 = (float*)(O + o_a);
  d.b32 = (float*)(O + o_b);
  cudaStream_t st = b->st;
  CK(cudaMemsetAsync(O + o_zero, 0, kZeroBytes, st));
  CK(cudaMemsetAsync(O + o_a, 0, 4 * 768, st));
  CK(cudaMemsetAsync(O + o_b, 0, 4 * 768, st));
  CK(cudaMemcpyAsync(O + o_desc, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d.bin_count, gcount.data(), 4 * 256, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d.bin_start, gstart.data(), 4 * 257, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(O + o_srcoff, src_off.data(), 8 * (nsrc + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(O + o_srcm, src_m.data(), 8 * nsrc, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(O + o_srcbin, src_bin.data(), 4 * 257 * (size_t)nsrc, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(O + o_dstbin, dst_bin.data(), 4 * 256 * (size_t)nsrc, cudaMemcpyHostToDevice, st));
  RegroupTab rt;
  rt.nsrc = nsrc;
  rt.recv = d_recv;
  rt.src_off = (const long long*)(O + o_srcoff);
  rt.src_m = (const long long*)(O + o_srcm);
  rt.src_bin_off = (const unsigned*)(O + o_srcbin);
  rt.dst_bin_off = (const unsigned*)(O + o_dstbin);
  rt.total = M;
  const ImgDesc* dd = (const ImgDesc*)(O + o_desc);
  if (M > 0) {
    launch_fit_regroup(dd, rt, st);
    launch_fit_bins(dd, 1, max_seg_nodes(M), std::min(d.blas_threads, kMaxBlasThreads), st);
    c->launches += 5;
  }
  CK(cudaMemcpyAsync(h_a32, d.a32, 4 * 768, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_b32, d.b32, 4 * 768, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_status, d.status, 4, cudaMemcpyDeviceToHost, st));
  return sync_status(b);
}

}  // extern "C"

namespace {
void piece_bits(Band* b, uint64_t* h_bits) {
  uint8_t* D = (uint8_t*)b->tabs;
  cudaMemcpy(h_bits, D + b->sc_dct.bits, 8 * 3, cudaMemcpyDeviceToHost);
  cudaMemcpy(h_bits + 3, D + b->sc_pln.bits, 8 * 4, cudaMemcpyDeviceToHost);
}
}  // namespace

extern "C" {

int hdll_b200_band_code(hdll_b200_ctx* ctx, const float* h_a32, const float* h_b32, const int32_t* h_first,
                        uint32_t* h_crc, int64_t* h_cnt, int32_t* h_out_a, uint64_t* h_bits, uint64_t* h_piece_ptr) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_a32 || !h_b32 || !h_first || !h_crc || !h_cnt || !h_out_a || !h_bits || !h_piece_ptr)
    return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  const ImgDesc& d = b->desc;
  CK(cudaMemcpyAsync(d.a32, h_a32, 4 * 768, cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(d.b32, h_b32, 4 * 768, cudaMemcpyHostToDevice, b->st));
  launch_estimate(b->d_desc, 1, d.n, b->st);
  launch_crc(b->d_desc, 1, b->crc_units, b->st);
  c->launches += 3;
  CK(cudaMemcpyAsync(h_crc, d.crc, 4 * 5, cudaMemcpyDeviceToHost, b->st));
  // a piece that starts its chain is coded now from the reset state (count 0,
  // A = 4); the others only count their symbols per context
  std::vector<long long> zc(kPieces * kMaxCtx, 0);
  std::vector<int> a4(kPieces * kMaxCtx, 4);
  if (int rc = pieces_to_dev(b, b->sc_dct.in_cnt, b->sc_pln.in_cnt, zc.data())) return rc;
  if (int rc = pieces_to_dev(b, b->sc_dct.in_a, b->sc_pln.in_a, a4.data())) return rc;
  int modes[kPieces];
  for (int k = 0; k < kPieces; k++) modes[k] = h_first[k] ? 0 : 1;
  if (int rc = run_chains(c, b, modes)) return rc;
  if (int rc = pieces_from_dev(b, b->sc_dct.out_cnt, b->sc_pln.out_cnt, (long long*)h_cnt)) return rc;
  if (int rc = pieces_from_dev(b, b->sc_dct.out_a, b->sc_pln.out_a, (int*)h_out_a)) return rc;
  piece_bits(b, h_bits);
  for (int k = 0; k < kPieces; k++) h_piece_ptr[k] = (uint64_t)(uintptr_t)b->piece_ptr[k];
  unsigned s = 0;
  CK(cudaMemcpy(&s, d.status, 4, cudaMemcpyDeviceToHost));
  return map_status(s);
}

int hdll_b200_band_maps(hdll_b200_ctx* ctx, const int64_t* h_in_cnt, const int32_t* h_need, int64_t* h_maps) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_in_cnt || !h_need || !h_maps) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  if (int rc = pieces_to_dev(b, b->sc_dct.in_cnt, b->sc_pln.in_cnt, (const long long*)h_in_cnt)) return rc;
  int modes[kPieces];
  for (int k = 0; k < kPieces; k++) modes[k] = h_need[k] ? 2 : kModeSkip;
  if (int rc = run_chains(c, b, modes)) return rc;
  AMap m[kPieces * kMaxCtx];
  if (int rc = pieces_from_dev(b, b->sc_dct.out_map, b->sc_pln.out_map, m)) return rc;
  for (int i = 0; i < kPieces * kMaxCtx; i++) {
    h_maps[3 * i + 0] = m[i].c;
    h_maps[3 * i + 1] = m[i].s;
    h_maps[3 * i + 2] = m[i].t;
  }
  return HDLL_B200_OK;
}

int hdll_b200_band_emit(hdll_b200_ctx* ctx, const int64_t* h_in_cnt, const int32_t* h_in_a, const int32_t* h_emit,
                        uint64_t* h_bits, uint64_t* h_piece_ptr) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  Band* b = band_of(ctx);
  if (!b || !h_in_cnt || !h_in_a || !h_emit || !h_bits || !h_piece_ptr) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  for (int i = 0; i < kPieces * kMaxCtx; i++)
    if (h_in_a[i] < 0 || h_in_a[i] >= kADomain) return HDLL_B200_E_ARG;
  if (int rc = pieces_to_dev(b, b->sc_dct.in_cnt, b->sc_pln.in_cnt, (const long long*)h_in_cnt)) return rc;
  if (int rc = pieces_to_dev(b, b->sc_dct.in_a, b->sc_pln.in_a, (const int*)h_in_a)) return rc;
  int modes[kPieces];
  for (int k = 0; k < kPieces; k++) modes[k] = h_emit[k] ? 0 : kModeSkip;
  if (int rc = run_chains(c, b, modes)) return rc;
  piece_bits(b, h_bits);
  for (int k = 0; k < kPieces; k++) h_piece_ptr[k] = (uint64_t)(uintptr_t)b->piece_ptr[k];
  unsigned s = 0;
  CK(cudaMemcpy(&s, b->desc.status, 4, cudaMemcpyDeviceToHost));
  return map_status(s);
}

int hdll_b200_assemble_pieces(hdll_b200_ctx* ctx, const hdll_b200_image* img, const uint32_t* crc, const float* a32,
                              const float* b32, const uint32_t* hist, const int32_t* npieces,
                              const uint64_t* piece_ptr, const uint64_t* piece_bits, uint8_t* d_out, uint64_t cap,
                              uint64_t* d_len, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  if (!c || !img || !crc || !a32 || !b32 || !hist || !npieces || !piece_ptr || !piece_bits || !d_out || !d_len)
    return HDLL_B200_E_ARG;
  if (img->width == 0 || img->height == 0) return HDLL_B200_E_EMPTY;
  CK(cudaSetDevice(c->device));
  if (!c->band) c->band = new Band();
  Band* b = c->band;
  cudaStream_t st = (cudaStream_t)stream;
  int np = 0;
  unsigned long long chain_bits[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k < 5; k++) {
    if (npieces[k] < 0) return HDLL_B200_E_ARG;
    for (int j = 0; j < npieces[k]; j++) chain_bits[k] += piece_bits[np + j];
    np += npieces[k];
  }
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  size_t o_chain[5];
  for (int k = 0; k < 5; k++) o_chain[k] = take((chain_bits[k] + 31) / 32 * 4 + 16);
  const size_t o_desc = take(sizeof(ImgDesc)), o_zero = take(kZeroBytes), o_crc = take(4 * 8);
  const size_t o_a = take(4 * 768), o_b = take(4 * 768), o_pre = take(img->hdr_pre_len + 1);
  const size_t o_post = take(img->hdr_post_len + 1), o_ptr = take(8 * (size_t)np), o_dbit = take(8 * (size_t)np);
  const size_t o_nbit = take(8 * (size_t)np), o_at = take(8 * 10), o_hist = take(4 * 256);
  if (ensure(&b->asmb, &b->asmb_cap, o, true)) return HDLL_B200_E_CUDA;
  uint8_t* A = (uint8_t*)b->asmb;
  std::vector<unsigned long long> dbit(np);
  np = 0;
  for (int k = 0; k < 5; k++) {
    unsigned long long run = 0;
    for (int j = 0; j < npieces[k]; j++) {
      dbit[np + j] = run;
      run += piece_bits[np + j];
    }
    np += npieces[k];
  }
  std::vector<const uint8_t*> ptrs(np);
  for (int i = 0; i < np; i++) ptrs[i] = (const uint8_t*)(uintptr_t)piece_ptr[i];
  CK(cudaMemsetAsync(A, 0, o_desc, st));  // the chains start zeroed (k_bitcat ORs)
  CK(cudaMemsetAsync(A + o_zero, 0, kZeroBytes, st));
  CK(cudaMemcpyAsync(A + o_ptr, ptrs.data(), 8 * (size_t)np, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_dbit, dbit.data(), 8 * (size_t)np, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_nbit, piece_bits, 8 * (size_t)np, cudaMemcpyHostToDevice, st));
  np = 0;
  for (int k = 0; k < 5; k++) {
    unsigned long long mx = 0;
    for (int j = 0; j < npieces[k]; j++) mx = std::max(mx, (unsigned long long)piece_bits[np + j]);
    launch_bitcat(A + o_chain[k], (const uint8_t* const*)(A + o_ptr) + np,
                  (const unsigned long long*)(A + o_dbit) + np, (const unsigned long long*)(A + o_nbit) + np,
                  npieces[k], mx, st);
    np += npieces[k];
  }
  // assembly desc: the full image's geometry, table, CRCs and headers
  ImgDesc d;
  memset(&d, 0, sizeof(d));
  d.w = (int)img->width;
  d.h = (int)img->height;
  d.n = (long long)d.w * d.h;
  d.slrme = img->params.slrme;
  d.status = (unsigned*)(A + o_zero + 8);
  d.bin_count = (unsigned*)(A + o_hist);
  d.crc = (unsigned*)(A + o_crc);
  d.a32 = (float*)(A + o_a);
  d.b32 = (float*)(A + o_b);
  d.hdr_pre = A + o_pre;
  d.hdr_pre_len = (int)img->hdr_pre_len;
  d.hdr_post = A + o_post;
  d.hdr_post_len = (int)img->hdr_post_len;
  d.out = d_out;
  d.out_len = (unsigned long long*)d_len;
  d.out_cap = (long long)cap;
  CK(cudaMemcpyAsync(A + o_hist, hist, 4 * 256, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_crc, crc, 4 * 5, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_a, a32, 4 * 768, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_b, b32, 4 * 768, cudaMemcpyHostToDevice, st));
  if (img->hdr_pre_len) CK(cudaMemcpyAsync(A + o_pre, img->hdr_pre, img->hdr_pre_len, cudaMemcpyHostToDevice, st));
  if (img->hdr_post_len) CK(cudaMemcpyAsync(A + o_post, img->hdr_post, img->hdr_post_len, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(A + o_desc, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  // AsmTab arrays: dct_out[1], dct_bits[1], plane_out[4], plane_bits[4]
  uint64_t at_h[10];
  at_h[0] = (uint64_t)(uintptr_t)(A + o_chain[0]);
  at_h[1] = chain_bits[0];
  for (int k = 0; k < 4; k++) {
    at_h[2 + k] = (uint64_t)(uintptr_t)(A + o_chain[1 + k]);
    at_h[6 + k] = chain_bits[1 + k];
  }
  CK(cudaMemcpyAsync(A + o_at, at_h, sizeof(at_h), cudaMemcpyHostToDevice, st));
  AsmTab at;
  at.dct_out = (uint8_t* const*)(A + o_at);
  at.dct_bits = (const unsigned long long*)(A + o_at + 8);
  at.plane_out = (uint8_t* const*)(A + o_at + 16);
  at.plane_bits = (const unsigned long long*)(A + o_at + 48);
  launch_assemble((const ImgDesc*)(A + o_desc), 1, at, (long long)cap, st);
  c->launches = 6;
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  unsigned s = 0;
  CK(cudaMemcpy(&s, d.status, 4, cudaMemcpyDeviceToHost));
  return map_status(s);
}

}  // extern "C"
