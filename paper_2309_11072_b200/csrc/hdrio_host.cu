// hdrio_host.cu -- C ABI of the .hdr scanline coder (include/hdll_b200.h
// hdll_b200_hdr_*), host side of hdrio.cu.
//
// Reading: a walk over the scanlines that only hops packet headers validates
// every new-RLE scanline exactly as radiance_io.py:167-215 does and records
// where each component stream starts; the device expands the packets.  A file
// with any flat / old-RLE scanline (radiance_io.py:218-242, whose repeat
// markers carry the previous pixel across scanlines) is expanded by this host
// loop instead and uploaded.
#include <vector>

#include "host_common.cuh"

using namespace hdll;
using namespace hdll_host;

namespace {

constexpr int kMinRleWidth = 8, kMaxRleWidth = 0x7FFF;  // radiance_io.py _MIN/_MAX_RLE_WIDTH

// the whole binary part on the host (flat / old-RLE present): radiance_io.py:157-242
int decode_host(const uint8_t* d, uint64_t len, int w, int h, uint8_t* out, uint64_t* used, int64_t* detail) {
  uint64_t pos = 0;
  bool have_prev = false;
  uint8_t prev[4] = {0, 0, 0, 0};
  for (int y = 0; y < h; y++) {
    uint8_t* row = out + (size_t)y * w * 4;
    if (w >= kMinRleWidth && w <= kMaxRleWidth && pos + 4 <= len && d[pos] == 2 && d[pos + 1] == 2 &&
        (d[pos + 2] & 0x80) == 0) {
      const int length = (d[pos + 2] << 8) | d[pos + 3];
      if (length != w) {
        detail[0] = length;
        detail[1] = w;
        return HDLL_B200_HDR_LENGTH;
      }
      pos += 4;
      for (int c = 0; c < 4; c++) {
        int j = 0;
        while (j < w) {
          if (pos >= len) return HDLL_B200_HDR_TRUNC_LINE;
          const int code = d[pos++];
          if (code > 128) {
            const int run = code & 0x7F;
            if (pos >= len) return HDLL_B200_HDR_TRUNC_RUN;
            if (j + run > w) return HDLL_B200_HDR_RUN_OVERFLOW;
            for (int k = 0; k < run; k++) row[4 * (j + k) + c] = d[pos];
            pos++;
            j += run;
          } else {
            if (code == 0) return HDLL_B200_HDR_ZERO_LITERAL;
            if (j + code > w) return HDLL_B200_HDR_LIT_OVERFLOW;
            if (pos + code > len) return HDLL_B200_HDR_TRUNC_LIT;
            for (int k = 0; k < code; k++) row[4 * (j + k) + c] = d[pos + k];
            pos += code;
            j += code;
          }
        }
      }
      memcpy(prev, row + 4 * (size_t)(w - 1), 4);
      have_prev = true;
      continue;
    }
    int j = 0, rshift = 0;
    while (j < w) {
      if (pos + 4 > len) return HDLL_B200_HDR_TRUNC_DATA;
      const uint8_t r = d[pos], g = d[pos + 1], b = d[pos + 2], e = d[pos + 3];
      pos += 4;
      if (r == 1 && g == 1 && b == 1) {  // repeat marker
        if (!have_prev) return HDLL_B200_HDR_REPEAT_FIRST;
        const long long count = (long long)e << rshift;
        if (j + count > w) return HDLL_B200_HDR_REPEAT_OVERFLOW;
        for (long long k = 0; k < count; k++) memcpy(row + 4 * (j + k), prev, 4);
        j += (int)count;
        rshift += 8;
      } else {
        uint8_t* px = row + 4 * (size_t)j;
        px[0] = r, px[1] = g, px[2] = b, px[3] = e;
        memcpy(prev, px, 4);
        have_prev = true;
        j++;
        rshift = 0;
      }
    }
  }
  *used = pos;
  return HDLL_B200_OK;
}

}  // namespace

extern "C" {

int hdll_b200_hdr_decode(hdll_b200_ctx* ctx, const uint8_t* h_data, uint64_t len, uint32_t width, uint32_t height,
                         uint8_t* d_rgbe, uint64_t* h_consumed, int64_t* h_detail, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  if (!c || (!h_data && len) || !d_rgbe || !h_consumed || !h_detail || width == 0 || height == 0)
    return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int w = (int)width, h = (int)height;
  // walk: every scanline new-RLE? record the component stream starts
  std::vector<long long> starts(4 * (size_t)h);
  uint64_t pos = 0;
  bool all_new = w >= kMinRleWidth && w <= kMaxRleWidth;
  for (int y = 0; y < h && all_new; y++) {
    const uint8_t* d = h_data;
    if (!(pos + 4 <= len && d[pos] == 2 && d[pos + 1] == 2 && (d[pos + 2] & 0x80) == 0)) {
      all_new = false;
      break;
    }
    const int length = (d[pos + 2] << 8) | d[pos + 3];
    if (length != w) {
      h_detail[0] = length;
      h_detail[1] = w;
      return HDLL_B200_HDR_LENGTH;
    }
    pos += 4;
    for (int cc = 0; cc < 4; cc++) {
      starts[4 * (size_t)y + cc] = (long long)pos;
      int j = 0;
      while (j < w) {
        if (pos >= len) return HDLL_B200_HDR_TRUNC_LINE;
        const int code = d[pos++];
        if (code > 128) {
          const int run = code & 0x7F;
          if (pos >= len) return HDLL_B200_HDR_TRUNC_RUN;
          if (j + run > w) return HDLL_B200_HDR_RUN_OVERFLOW;
          pos++;
          j += run;
        } else {
          if (code == 0) return HDLL_B200_HDR_ZERO_LITERAL;
          if (j + code > w) return HDLL_B200_HDR_LIT_OVERFLOW;
          if (pos + code > len) return HDLL_B200_HDR_TRUNC_LIT;
          pos += code;
          j += code;
        }
      }
    }
  }
  if (!all_new) {  // flat / old-RLE scanlines: the host decodes the file
    std::vector<uint8_t> rgbe(4 * (size_t)w * h);
    uint64_t used = 0;
    const int rc = decode_host(h_data, len, w, h, rgbe.data(), &used, h_detail);
    if (rc) return rc;
    CK(cudaMemcpyAsync(d_rgbe, rgbe.data(), rgbe.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    *h_consumed = used;
    return HDLL_B200_OK;
  }
  // device: the scanline bytes, the starts, the new-RLE flags
  const size_t o_data = 0, o_starts = align_up(pos + 16), o_flags = align_up(o_starts + 8 * starts.size());
  const size_t need = align_up(o_flags + (size_t)h);
  if (ensure(&c->hdr_buf, &c->hdr_cap, need, true)) return HDLL_B200_E_CUDA;
  uint8_t* D = (uint8_t*)c->hdr_buf;
  std::vector<uint8_t> flags((size_t)h, 1);
  CK(cudaMemcpyAsync(D + o_data, h_data, pos, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(D + o_starts, starts.data(), 8 * starts.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(D + o_flags, flags.data(), flags.size(), cudaMemcpyHostToDevice, st));
  launch_hdr_expand(D + o_data, (const long long*)(D + o_starts), D + o_flags, w, h, d_rgbe, st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  *h_consumed = pos;
  return HDLL_B200_OK;
}

int hdll_b200_hdr_encode(hdll_b200_ctx* ctx, const uint8_t* d_rgbe, uint32_t width, uint32_t height, int32_t rle,
                         uint8_t* h_out, uint64_t cap, uint64_t* h_len, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  CtxLock lock(c);
  if (!c || !d_rgbe || !h_out || !h_len || width == 0 || height == 0) return HDLL_B200_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int w = (int)width, h = (int)height;
  if (!(rle && w >= kMinRleWidth && w <= kMaxRleWidth)) {  // flat scanlines
    const uint64_t n = 4ULL * w * h;
    *h_len = n;
    if (n > cap) return HDLL_B200_E_CAPACITY;
    CK(cudaMemcpyAsync(h_out, d_rgbe, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HDLL_B200_OK;
  }
  const size_t n4 = 4 * (size_t)h;
  const size_t max_bytes = (size_t)h * (4 + 4 * ((size_t)w + (w + 127) / 128));
  const size_t o_sizes = 0, o_offs = align_up(8 * n4), o_out = align_up(o_offs + 8 * n4);
  if (ensure(&c->hdr_buf, &c->hdr_cap, o_out + max_bytes + 16, true)) return HDLL_B200_E_CUDA;
  uint8_t* D = (uint8_t*)c->hdr_buf;
  launch_hdr_sizes(d_rgbe, w, h, (long long*)(D + o_sizes), st);
  std::vector<long long> sz(n4), offs(n4);
  CK(cudaMemcpyAsync(sz.data(), D + o_sizes, 8 * n4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  long long run = 0;
  for (int y = 0; y < h; y++) {
    run += 4;  // 2 2 hi lo
    for (int cc = 0; cc < 4; cc++) {
      offs[4 * (size_t)y + cc] = run;
      run += sz[4 * (size_t)y + cc];
    }
  }
  *h_len = (uint64_t)run;
  if ((uint64_t)run > cap) return HDLL_B200_E_CAPACITY;
  CK(cudaMemcpyAsync(D + o_offs, offs.data(), 8 * n4, cudaMemcpyHostToDevice, st));
  launch_hdr_write(d_rgbe, w, h, (const long long*)(D + o_offs), D + o_out, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_out, D + o_out, (size_t)run, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HDLL_B200_OK;
}

}  // extern "C"
