// hdrio.cu -- Radiance .hdr scanline coding on the GPU (
// reference radiance_io.py:119-317).
//
// Writing (write_hdr, radiance_io.py:245-317): every scanline of width in
// [8, 32767] becomes `2 2 hi lo` and four per-component packet streams
// (_encode_component: maximal runs of >= 4 equal bytes as run packets of
// <= 127, the bytes between as literal packets of <= 128).  Scanlines are
// independent: one thread per (scanline, component) sizes its packets, a scan
// over the scanlines places them, the same threads write them.
//
// Reading (parse_hdr, radiance_io.py:119-242): a new-RLE scanline's component
// streams follow one another, so their starts are found by a host walk that
// only hops packet headers (csrc/api.cu hdll_b200_hdr_decode); one thread per
// (scanline, component) then expands its packets.  Flat / old-RLE scanlines
// (which may repeat the previous scanline's last pixel) are expanded by the
// same host walk.
#include "encoder.cuh"

namespace hdll {

constexpr int kHdrMinRun = 4;  // radiance_io.py _MIN_RUN

// Packet bytes of one component of one scanline, and (if out) the packets.
// vals(x) is the component's byte at pixel x.
template <class V>
__device__ long long encode_component(const V& vals, int n, uint8_t* out) {
  long long o = 0;
  auto literals = [&](int start, int end) {  // _flush_literals
    while (start < end) {
      const int chunk = min(end - start, 128);
      if (out) {
        out[o] = (uint8_t)chunk;
        for (int i = 0; i < chunk; i++) out[o + 1 + i] = vals(start + i);
      }
      o += 1 + chunk;
      start += chunk;
    }
  };
  int lit_start = 0, s = 0;
  while (s < n) {  // maximal runs [s, e) of one value
    const uint8_t v = vals(s);
    int e = s + 1;
    while (e < n && vals(e) == v) e++;
    if (e - s >= kHdrMinRun) {
      literals(lit_start, s);
      int length = e - s;
      while (length > 0) {
        const int chunk = min(length, 127);
        if (out) {
          out[o] = (uint8_t)(0x80 | chunk);
          out[o + 1] = v;
        }
        o += 2;
        length -= chunk;
      }
      lit_start = e;
    }
    s = e;
  }
  literals(lit_start, n);
  return o;
}

struct RowComp {
  const uint8_t* row;  // (w, 4) RGBE of the scanline
  int c;
  __device__ __forceinline__ uint8_t operator()(int x) const { return row[4 * x + c]; }
};

// pass 1: bytes of every (scanline, component); sizes[y * 4 + c]
__global__ void __launch_bounds__(128) k_hdr_sizes(const uint8_t* __restrict__ rgbe, int w, int h, long long* sizes) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4LL * h) return;
  const int y = (int)(i >> 2), c = (int)(i & 3);
  sizes[i] = encode_component(RowComp{rgbe + (long long)y * w * 4, c}, w, nullptr);
}

// pass 2 (after the host scan): offs[y * 4 + c] = where the packets go
__global__ void __launch_bounds__(128) k_hdr_write(const uint8_t* __restrict__ rgbe, int w, int h,
                                                   const long long* offs, uint8_t* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4LL * h) return;
  const int y = (int)(i >> 2), c = (int)(i & 3);
  uint8_t* o = out + offs[i];
  if (c == 0) {  // the scanline header 2 2 hi lo sits before component 0
    o[-4] = 2;
    o[-3] = 2;
    o[-2] = (uint8_t)(w >> 8);
    o[-1] = (uint8_t)(w & 0xFF);
  }
  encode_component(RowComp{rgbe + (long long)y * w * 4, c}, w, o);
}

// read: expand the packets of one (scanline, component) whose stream starts at
// starts[y * 4 + c] (validated by the host walk)
__global__ void __launch_bounds__(128) k_hdr_expand(const uint8_t* __restrict__ data, const long long* starts,
                                                    const uint8_t* newrle, int w, int h, uint8_t* rgbe) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4LL * h) return;
  const int y = (int)(i >> 2), c = (int)(i & 3);
  if (!newrle[y]) return;
  const uint8_t* p = data + starts[i];
  uint8_t* row = rgbe + (long long)y * w * 4 + c;
  int j = 0;
  while (j < w) {
    const int code = *p++;
    if (code > 128) {
      const int run = code & 0x7F;
      const uint8_t v = *p++;
      for (int k = 0; k < run; k++) row[4 * (j + k)] = v;
      j += run;
    } else {
      for (int k = 0; k < code; k++) row[4 * (j + k)] = p[k];
      p += code;
      j += code;
    }
  }
}

void launch_hdr_sizes(const uint8_t* rgbe, int w, int h, long long* sizes, cudaStream_t st) {
  k_hdr_sizes<<<(unsigned)((4LL * h + 127) / 128), 128, 0, st>>>(rgbe, w, h, sizes);
}

void launch_hdr_write(const uint8_t* rgbe, int w, int h, const long long* offs, uint8_t* out, cudaStream_t st) {
  k_hdr_write<<<(unsigned)((4LL * h + 127) / 128), 128, 0, st>>>(rgbe, w, h, offs, out);
}

void launch_hdr_expand(const uint8_t* data, const long long* starts, const uint8_t* newrle, int w, int h,
                       uint8_t* rgbe, cudaStream_t st) {
  k_hdr_expand<<<(unsigned)((4LL * h + 127) / 128), 128, 0, st>>>(data, starts, newrle, w, h, rgbe);
}

}  // namespace hdll
