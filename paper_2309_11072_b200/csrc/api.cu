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
#include "host_common.cuh"

using namespace hdll;
using namespace hdll_host;

namespace {

// The per-batch staging block (descriptors, parameters, chain tables) lives in
// pinned host memory; this kernel pulls it over PCIe itself instead of a
// cudaMemcpyAsync, which would queue on the copy engine behind any large
// host->device transfer in flight (the next chunk's RGBE in HostPipeline) and
// stall the whole batch.  It also zeroes every image's small reset block.
constexpr int kMaxZero = 256;
__global__ void __launch_bounds__(256) k_stage(uint8_t* dst, const uint8_t* src, size_t bytes,
                                               uint8_t* const* zp, int nz) {
  __shared__ uint8_t* zs[kMaxZero];
  for (int i = threadIdx.x; i < nz; i += blockDim.x) zs[i] = zp[i];
  __syncthreads();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (long long i = tid; i < (long long)(bytes / 16); i += stride) d4[i] = s4[i];
  constexpr int zq = (int)(kZeroBytes / 16);
  for (long long j = tid; j < (long long)nz * zq; j += stride)
    reinterpret_cast<uint4*>(zs[j / zq])[j % zq] = make_uint4(0, 0, 0, 0);
}
static_assert(kZeroBytes % 16 == 0, "reset blocks are zeroed in 16-byte words");

// stage `bytes` of H (pinned) into D and zero the reset blocks at zp[0..nz)
int stage_upload(uint8_t* D, const uint8_t* H, size_t bytes, uint8_t* const* zp, int nz, cudaStream_t st) {
  for (int z0 = 0; z0 < nz || z0 == 0; z0 += kMaxZero) {
    const int cnt = std::min(kMaxZero, nz - z0);
    const size_t b = z0 == 0 ? bytes : 0;
    long long blocks = (long long)(b / 16 + cnt * (kZeroBytes / 16) + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    if (blocks < 1) blocks = 1;
    k_stage<<<(unsigned)blocks, 256, 0, st>>>(D, H, b, zp + z0, cnt < 0 ? 0 : cnt);
    if (nz == 0) break;
  }
  return cuda_fail(cudaGetLastError(), "stage");
}

// DCT coder lanes code runs of kDctMaxBlocksPerLane consecutive blocks: a
// tile's fixed cost (three look-backs, the warp scans of counts and A-maps,
// the release stores) is spread over 4x the symbols.  Measured against 1 and
// 2 blocks per lane (and 8, which needs more shared memory): 4 is fastest on
// config 1 (entropy_dct 2.85 -> 2.04 ms), config 3 (1.55 -> 0.75 ms) and even
// the single 4096x2160 image of config 2 (0.42 -> 0.23 ms).
int dct_blocks_per_lane() {
#ifdef HDLL_DCT_BPL  // experiment builds: a fixed value
  return HDLL_DCT_BPL;
#endif
  return kDctMaxBlocksPerLane;
}

// mode: 0 full encode, 1 lossless plane (rgbe -> plane bytes), 2 lossy image (rgbe -> sdr rgb)
int run_batch(Ctx* c, const hdll_b200_image* imgs, int n, uint8_t* const* d_out, const uint64_t* out_cap,
              uint64_t* d_out_len, cudaStream_t st, int mode) {
  if (n <= 0) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  // the arena, tables and status area are reused: a batch on another stream
  // waits for the previous batch on the device
  if (c->done_ev && c->last_stream != st) CK(cudaStreamWaitEvent(st, c->done_ev, 0));
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
  size_t stage_bytes = 0;
  for (int i = 0; i < n; i++) stage_bytes += params_stage_bytes(imgs[i]);
  // sequential-coder chains: the DCT stream of every image (kind 0) and its 4
  // plane streams (kinds 1..4), each family driven by its own kernel
  HostChains hc_dct, hc_pln;
  {
    long long rows = 0;
    int mw = 1;
    for (int i = 0; i < n; i++) {
      rows += (mode == 0 ? 4 : (mode == 1 ? 1 : 0)) * (long long)imgs[i].height;
      mw = std::max(mw, (int)imgs[i].width);
    }
    hc_pln.segw = plane_segw_for(rows, mw);
  }
  // A full encode codes each image's base layer as two chains: Y (contexts
  // 0-2) and Cb, Cr (contexts 3-5).  No state crosses between them -- the
  // reference's shared A/N arrays keep Y's and the chroma's contexts apart --
  // so twice as many chains share the GPU, and the assembly appends the
  // chroma bits to the Y bits.
  const bool dct_split = mode == 0;
  hc_dct.dct_bpl = dct_blocks_per_lane();
  for (int i = 0; i < n; i++) {
    const long long w = imgs[i].width, h = imgs[i].height;
    const long long nb = ((w + 7) / 8) * ((h + 7) / 8);
    for (int k = 0; k < 5; k++) {
      bool active = (mode == 0) || (mode == 1 && k == 1) || (mode == 2 && k == 0);
      uint8_t* out = A + base[i] + lays[i].off_chain[k];
      if (k == 0 && dct_split) {
        const long long ycap = dct_y_cap(nb);
        hc_dct.add(i, 0, 0, 0, nb, out, ycap, (int)w);
        hc_dct.add(i, 0, -2, 0, nb, out + ycap, lays[i].chain_cap[0] - ycap, (int)w);
        continue;
      }
      (k == 0 ? hc_dct : hc_pln).add(i, k, -1, 0, active ? (k == 0 ? nb : h) : 0, out, lays[i].chain_cap[k], (int)w);
    }
  }
  hc_dct.schedule();
  hc_pln.schedule();
  const long long ntiles = hc_dct.ntiles() + hc_pln.ntiles();
  size_t tab_bytes = align_up(sizeof(ImgDesc) * n) + hc_dct.staged_bytes() + hc_pln.staged_bytes() + 16 * kAlign +
                     align_up(8 * (size_t)n);
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
  const size_t t_zero = stage(nullptr, 8 * (size_t)n);  // read by k_stage from the pinned block itself
  uint8_t** zero_ptrs = reinterpret_cast<uint8_t**>(H + t_zero);

  long long max_n = 0, max_sort_tiles = 0, max_nodes = 0, max_out = 0;
  int max_w = 0, max_h = 0, max_radius = 0, max_level = 0, max_base_tiles = 0, max_chunks = 1;
  bool any_real = false, any_slrme = false, any_non3 = false, any_hist = false, any_int = false, any_sortfit = false;
  for (int i = 0; i < n; i++) {
    const auto& im = imgs[i];
    const auto& p = im.params;
    const ImgLayout& L = lays[i];
    uint8_t* B = A + base[i];
    ImgDesc& d = ds[i];
    const StagedParams sp = stage_params(stage, im);
    fill_desc(d, im, L, B, mode, any_trace, D, sp);
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
    any_non3 |= (d.slrme && d.sigma_milli != 0 && d.radius != 3);
    any_slrme |= d.slrme != 0;
    any_hist |= (d.slrme && !d.fit_owner && !d.hist_fused);
    any_int |= d.int_fit != 0;
    any_sortfit |= (d.slrme && !d.int_fit);
  }
  const long long crc_units = crc_assign_units(ds.data(), n);
  memcpy(H + t_descs, ds.data(), sizeof(ImgDesc) * n);
  memset(H + t_ticket, 0, 16);
  for (int i = 0; i < n; i++) zero_ptrs[i] = A + base[i] + lays[i].off_zero;
  if (int rc = stage_upload(D, H, so, zero_ptrs, n, st)) return rc;
  c->d_descs = (ImgDesc*)(D + t_descs);
  const ImgDesc* dd = c->d_descs;

  // entropy status arena
  if (int rc = prepare_estat(c, ntiles, st)) return rc;
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
    launch_base_layer(dd, n, max_base_tiles, max_n, st);
    c->launches += 3;
  }
  mark(kStBase);
  if (mode == 0 && any_real) {
    launch_prefilter(dd, n, max_w, max_h, max_radius, st, any_non3);
    c->launches += any_non3 ? 2 : 1;
  }
  mark(kStPrefilter);
  if (mode == 0 && any_sortfit) {  // sigma > 0: the order-replicating sums
    launch_fit(dd, n, (int)max_sort_tiles, max_nodes, max_chunks, st, any_hist);
    c->launches += any_hist ? 7 : 6;
  } else if (mode == 0 && any_hist) {  // bin counts of sigma-0 global-regression images
    launch_fit_hist(dd, n, (int)max_sort_tiles, st);
    c->launches += 1;
  }
  if (mode == 0 && any_int) {  // sigma = 0: exact integer bins
    launch_fit_int(dd, n, max_n, st);
    c->launches += 2;
  }
  mark(kStFit);
  if (mode == 0) {
    launch_estimate(dd, n, max_n, st);
    c->launches += 1;
  }
  mark(kStEstimate);
  launch_crc(dd, n, crc_units, st);
  c->launches += 2;
  mark(kStCrc);
  if (ct_dct.ntiles > 0) {
    if (ensure(&c->plane_scratch, &c->plane_scratch_cap,
               std::max(dct_scratch_bytes(ct_dct), plane_scratch_bytes(ct_pln, max_w)), true))
      return HDLL_B200_E_CUDA;
    launch_entropy_dct(dd, ct_dct, c->plane_scratch, st);
    launch_entropy_fixup(ct_dct, st);
    c->launches += 2;
  }
  mark(kStEntropyDct);
  if (ct_pln.ntiles > 0) {
    if (ensure(&c->plane_scratch, &c->plane_scratch_cap, plane_scratch_bytes(ct_pln, max_w), true))
      return HDLL_B200_E_CUDA;
    launch_entropy_plane(dd, ct_pln, max_w, c->plane_scratch, st);
    launch_entropy_fixup(ct_pln, st);
    c->launches += 2;
  }
  mark(kStEntropyPlane);
  if (mode == 0) {
    AsmTab at;
    at.dct_out = ct_dct.out;
    at.dct_bits = ct_dct.bits;
    at.dct_stride = dct_split ? 2 : 1;
    at.dct_split = dct_split;
    at.plane_out = ct_pln.out;
    at.plane_bits = ct_pln.bits;
    at.err_acc = c->err_acc;
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

// which coder bodies a decode job reads: sdr_only 0 all five, 1 the base layer
// (decode_sdr), 2 body 1 alone as a lossless plane (the plane coder plugin)
inline bool dec_uses(const hdll_b200_decode_image& di, int k) {
  return di.sdr_only == 0 || (di.sdr_only == 1 && k == 0) || (di.sdr_only == 2 && k == 1);
}

// GPU decode of a batch (decode.cu); synchronous.
int run_decode(Ctx* c, const hdll_b200_decode_image* imgs, int n, uint8_t* const* d_out, uint32_t* h_status,
               cudaStream_t st) {
  if (n <= 0) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  if (c->done_ev) CK(cudaEventSynchronize(c->done_ev));  // an encode batch may still use the arena
  c->launches = 0;
  // each image as the encoder's descriptor (same arena layout), plus its coder bodies
  std::vector<hdll_b200_image> ims(n);
  std::vector<ImgLayout> lays(n);
  std::vector<size_t> base(n);
  size_t total = 0;
  for (int i = 0; i < n; i++) {
    const auto& di = imgs[i];
    if (di.width == 0 || di.height == 0) return HDLL_B200_E_EMPTY;
    if (di.quality < 1 || di.quality > 100 || di.sigma_milli < 0 || di.radius < 0) return HDLL_B200_E_ARG;
    if (!di.sdr_only && di.slrme && di.sigma_milli && (!di.taps || di.radius < 1)) return HDLL_B200_E_ARG;
    if (di.sdr_only < 0 || di.sdr_only > 2) return HDLL_B200_E_ARG;
    hdll_b200_image& im = ims[i];
    memset(&im, 0, sizeof(im));
    im.width = di.width;
    im.height = di.height;
    im.params.quality = di.quality;
    im.params.sigma_milli = di.sigma_milli;
    im.params.slrme = di.slrme;
    im.params.blas_threads = 1;
    im.params.radius = di.radius;
    im.params.taps = di.taps;
    lays[i] = plan(im, false);
    base[i] = total;
    total += lays[i].total;
    for (int k = 0; k < 5; k++) total = align_up(total + (dec_uses(di, k) ? di.body_len[k] : 0) + 16);
  }
  if (ensure(&c->arena, &c->arena_cap, total, true)) return HDLL_B200_E_CUDA;
  uint8_t* A = (uint8_t*)c->arena;
  size_t stage_bytes = align_up(sizeof(ImgDesc) * n) + 4 * kAlign;
  for (int i = 0; i < n; i++) stage_bytes += params_stage_bytes(ims[i]) + 2 * align_up(4 * 768);
  const int slot = c->slot;
  c->slot ^= 1;
  if (c->slot_ev[slot]) CK(cudaEventSynchronize(c->slot_ev[slot]));
  else CK(cudaEventCreateWithFlags(&c->slot_ev[slot], cudaEventDisableTiming));
  if (ensure(&c->pinned_slot[slot], &c->pinned_cap_slot[slot], stage_bytes + 4096, false)) return HDLL_B200_E_CUDA;
  if (ensure(&c->tabs_slot[slot], &c->tabs_cap_slot[slot], stage_bytes + 4096, true)) return HDLL_B200_E_CUDA;
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
  std::vector<ImgDesc> ds(n);
  long long max_n = 0;
  int max_w = 0, max_h = 0, max_radius = 0, max_base_tiles = 0;
  bool any_real = false, all_sdr = true;
  for (int i = 0; i < n; i++) {
    const auto& di = imgs[i];
    uint8_t* B = A + base[i];
    const StagedParams sp = stage_params(stage, ims[i]);
    ImgDesc& d = ds[i];
    fill_desc(d, ims[i], lays[i], B, 0, false, D, sp);
    d.decode = 1;
    d.hist_fused = 0;
    d.slrme = di.sdr_only ? 0 : di.slrme;
    d.crc_mask = di.sdr_only == 1 ? 0x1 : (di.sdr_only == 2 ? 0x2 : 0x1F);
    d.out_rgbe = d_out[i];
    d.a32 = (float*)(D + stage(di.a32, 4 * 768));
    d.b32 = (float*)(D + stage(di.b32, 4 * 768));
    size_t o = base[i] + lays[i].total;
    for (int k = 0; k < 5; k++) {
      const size_t len = dec_uses(di, k) ? di.body_len[k] : 0;
      d.pay[k] = A + o;
      d.pay_bytes[k] = (long long)len;
      if (len) CK(cudaMemcpyAsync(A + o, di.body[k], len, cudaMemcpyHostToDevice, st));
      o = align_up(o + len + 16);
    }
    max_n = std::max(max_n, d.n);
    max_w = std::max(max_w, d.w);
    max_h = std::max(max_h, d.h);
    max_radius = std::max(max_radius, d.radius);
    max_base_tiles = std::max(max_base_tiles, (d.nbx + 15) / 16 * d.nby);
    any_real |= d.slrme && d.sigma_milli;
    all_sdr &= di.sdr_only == 1;
  }
  const long long crc_units = crc_assign_units(ds.data(), n);
  memcpy(H + t_descs, ds.data(), sizeof(ImgDesc) * n);
  CK(cudaMemcpyAsync(D, H, so, cudaMemcpyHostToDevice, st));
  for (int i = 0; i < n; i++) {
    CK(cudaMemsetAsync(A + base[i] + lays[i].off_zero, 0, kZeroBytes, st));
    CK(cudaMemsetAsync(ds[i].zz, 0, sizeof(int16_t) * 3 * ds[i].nblocks * 64, st));
  }
  const ImgDesc* dd = (const ImgDesc*)(D + t_descs);
  if (!all_sdr && 8LL * ((max_w + 4) & ~3) + 2048 > 227 * 1024) return HDLL_B200_E_ARG;  // planes wider than ~28.8k samples
  launch_decode_coders(dd, n, !all_sdr, max_w, st);
  launch_reconstruct(dd, n, max_base_tiles, st);
  c->launches += 2;
  if (any_real) {
    launch_prefilter(dd, n, max_w, max_h, max_radius, st);
    c->launches += 1;
  }
  launch_decode_output(dd, n, max_n, st);
  launch_crc(dd, n, crc_units, st);
  c->launches += 3;
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->slot_ev[slot], st));
  CK(cudaStreamSynchronize(st));
  c->dec_descs = ds;
  for (int i = 0; i < n; i++) {
    unsigned s = 0, crc[5] = {0, 0, 0, 0, 0};
    CK(cudaMemcpy(&s, ds[i].status, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(crc, ds[i].crc, sizeof(crc), cudaMemcpyDeviceToHost));
    uint32_t out = (s >> 16) & 0x1F;                    // stream k failed to decode
    if (s & (1u << 21)) out |= HDLL_B200_DEC_NO_ENTRY;  // exponent without a regression entry
    for (int k = 0; k < 5; k++)
      if (((ds[i].crc_mask >> k) & 1) && !((out >> k) & 1) && crc[k] != imgs[i].crc[k])
        out |= HDLL_B200_DEC_CRC << k;
    h_status[i] = out;
  }
  return HDLL_B200_OK;
}

// status of the last batch and of every encode batch since the previous
// check (the accumulated word is read and cleared)
int check_status(Ctx* c) {
  CK(cudaEventSynchronize(c->done_ev));
  unsigned worst = 0;
  for (auto& d : c->descs) {
    unsigned s = 0;
    CK(cudaMemcpy(&s, d.status, sizeof(s), cudaMemcpyDeviceToHost));
    worst |= s;
  }
  unsigned acc = 0;
  CK(cudaMemcpy(&acc, c->err_acc, sizeof(acc), cudaMemcpyDeviceToHost));
  if (acc) CK(cudaMemset(c->err_acc, 0, sizeof(acc)));
  return map_status(worst | acc);
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
  if (cudaMalloc(&c->err_acc, 256) != cudaSuccess || cudaMemset(c->err_acc, 0, 256) != cudaSuccess) {
    delete c;
    return HDLL_B200_E_CUDA;
  }
  upload_base_constants();
  upload_crc_constants();
  upload_fit_constants();
  upload_tonemap_constants();
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
  band_free(c);
  if (c->plane_scratch) cudaFree(c->plane_scratch);
  if (c->hdr_buf) cudaFree(c->hdr_buf);
  if (c->err_acc) cudaFree(c->err_acc);
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
  CtxLock lock(c);
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
  CtxLock lock(c);
  if (c->last_status) return c->last_status;
  if (!c->done_ev) return HDLL_B200_OK;
  return check_status(c);
}

int hdll_b200_encode_host(hdll_b200_ctx* ctx, const hdll_b200_image* img, uint8_t* h_out, uint64_t cap,
                          uint64_t* out_len) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !img || !h_out || !out_len) return HDLL_B200_E_ARG;
  CtxLock lock(c);
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
  if (!c || !h_dst) return HDLL_B200_E_ARG;
  CtxLock lock(c);
  const bool dec = (which & 16) != 0;  // the last decode batch (synchronous: already complete)
  which &= 15;
  const std::vector<ImgDesc>& dv = dec ? c->dec_descs : c->descs;
  if (index < 0 || index >= (int)dv.size() || (dec && which != 1 && which != 3)) return HDLL_B200_E_ARG;
  const ImgDesc& d = dv[index];
  if (!dec) CK(cudaEventSynchronize(c->done_ev));
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
  CtxLock lock(c);
  return plugin_common(c, h_plane, (size_t)w * h, w, h, 85, 1, h_body, cap, body_len, crc, nullptr);
}

int hdll_b200_lossy_encode(hdll_b200_ctx* ctx, const uint8_t* h_rgb, uint32_t w, uint32_t h, int32_t quality,
                           uint8_t* h_body, uint64_t cap, uint64_t* body_len, uint8_t* h_decoded, uint32_t* crc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !h_rgb || !h_body || !body_len || !crc || !h_decoded) return HDLL_B200_E_ARG;
  CtxLock lock(c);
  if (quality < 1 || quality > 100) return HDLL_B200_E_ARG;
  return plugin_common(c, h_rgb, (size_t)w * h * 3, w, h, quality, 2, h_body, cap, body_len, crc, h_decoded);
}

int hdll_b200_decode_batch(hdll_b200_ctx* ctx, const hdll_b200_decode_image* imgs, int n, uint8_t* const* d_out,
                           uint32_t* h_status, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !imgs || !d_out || !h_status) return HDLL_B200_E_ARG;
  CtxLock lock(c);
  return run_decode(c, imgs, n, d_out, h_status, (cudaStream_t)stream);
}

int hdll_b200_last_launch_count(hdll_b200_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  return c ? c->launches : 0;
}

int hdll_b200_stage_times(hdll_b200_ctx* ctx, float* ms, int n) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !ms || n < kStages || !c->stage_ev[0]) return HDLL_B200_E_ARG;
  CtxLock lock(c);
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
