// entropy.cu -- the two adaptive Golomb-Rice coders, parallelised.
//
// Reference (sequential, numba):
//   encode_plane          _kernels.py:169-216  (lossless coder id 1: MED + 5 contexts + runs)
//   encode_dct_component  _kernels.py:280-324  (base layer symbols, 6 contexts shared by Y/Cb/Cr,
//                                               codec_core.py:439-450)
//   _rice_put / _select_k / _update_state      _kernels.py:65-128
//
// Parallel form.  A *chain* is one sequential coder invocation (one DCT stream
// per image, one plane stream per (image, plane)); it is cut into *tiles*
// (a plane row, or 32 consecutive DCT blocks of one component), one warp per
// tile, lane = contiguous slice of the tile.  The symbols of a tile depend
// only on the data; the coder state carried between tiles is, per context,
// (count, A).  Each warp, in ONE pass with three chained decoupled look-backs
// (tiles are taken in order from an atomic ticket so every wait is on an
// already-running warp):
//   1. counts per context      -> look-back -> global symbol index of each symbol
//                                 (halving points and N follow from the index)
//   2. A-maps per context      -> look-back -> incoming A of the tile (common.cuh AMap)
//   3. code lengths            -> look-back -> bit offset of the tile in the chain
//   4. emit MSB-first bits straight into the chain's byte stream; words shared
//      between lanes are merged through a warp carry, the (at most two) words
//      a tile shares with its neighbours are parked and merged by the
//      k_entropy_fixup launch, so no warp ever waits on another's emission.
// Tickets are dealt round-robin over chains, so every chain advances at once.
// Flags carry the launch epoch, so status memory is never re-zeroed.
#include "encoder.cuh"

namespace hdll {

constexpr int kRunCtx = 4;  // _kernels.py:17

constexpr long long kSpinLimit = 1LL << 26;

__device__ __forceinline__ int wait_state(const ChainTab& ct, long long g, int which, unsigned* status) {
  const int* f = ct.flags + g * 4 + which;
  for (long long it = 0;; it++) {
    int v = ld_acquire(f);
    if ((v >> 2) == ct.epoch && (v & 3)) return v & 3;
    if (it > kSpinLimit) {
      atomicOr(status, kErrLookback);
      return 0;
    }
    __nanosleep(32);
  }
}

__device__ __forceinline__ void publish(const ChainTab& ct, long long g, int which, int state) {
  __threadfence();
  st_release(ct.flags + g * 4 + which, (ct.epoch << 2) | state);
}

// ---------------------------------------------------------------------------
// Bit emission with lane carry (see file comment).
// ---------------------------------------------------------------------------
struct WordSink {
  uint32_t* words;
  long long cap_words;
  long long tile_first_word;
  bool tile_start_partial;
  uint32_t* edge;  // this tile's [head, tail] slots
  unsigned* status;

  // complete words owned by this tile; the word it shares with the previous
  // tile (its first word when it starts mid-word) is parked in edge[0]
  __device__ void write(long long idx, uint32_t w) const {
    if (idx == tile_first_word && tile_start_partial) {
      edge[0] = w;
      return;
    }
    if (idx >= cap_words) {
      atomicOr(status, kErrCapacity);
      return;
    }
    words[idx] = __byte_perm(w, 0, 0x0123);  // MSB-first word -> stream byte order
  }
};

struct LaneBits {
  // streaming accumulator for one lane's bits starting at global bit s
  unsigned long long acc;
  int nacc;
  long long wpos;   // word index being filled
  long long first;  // first word index of the lane
  bool head_partial;
  bool have_head;
  uint32_t head;
  const WordSink* sink;

  __device__ void init(long long s, const WordSink* k) {
    sink = k;
    wpos = first = s >> 5;
    nacc = (int)(s & 31);
    acc = 0;
    head_partial = nacc != 0;
    have_head = false;
  }
  __device__ __forceinline__ void put(uint32_t bits, int len) {
    if (len == 0) return;
    acc = (acc << len) | (unsigned long long)bits;
    nacc += len;
    if (nacc >= 32) {
      uint32_t w = (uint32_t)(acc >> (nacc - 32));
      nacc -= 32;
      acc &= (nacc ? ((1ULL << nacc) - 1) : 0ULL);
      if (wpos == first && head_partial) {
        head = w;
        have_head = true;
      } else {
        sink->write(wpos, w);
      }
      wpos++;
    }
  }
};

// ---------------------------------------------------------------------------
// The tile engine (one warp).
// ---------------------------------------------------------------------------
template <int NCTX, class Gen>
__device__ void run_tile(const ChainTab& ct, int chain, long long tin, long long g, const Gen& gen, unsigned* status) {
  const int lane = threadIdx.x & 31;
  const bool chain_start = tin == 0;

  // ---- 1. counts ----
  int cnt[NCTX];
#pragma unroll
  for (int c = 0; c < NCTX; c++) cnt[c] = 0;
  gen.for_each([&](int ctx, int v, int xl, uint32_t xb) { cnt[ctx]++; });
  long long lbase[NCTX], tot[NCTX], incnt[NCTX];
#pragma unroll
  for (int c = 0; c < NCTX; c++) {
    long long t;
    lbase[c] = warp_excl_sum((long long)cnt[c], &t);
    tot[c] = t;
    incnt[c] = 0;
  }
  if (lane == 0) {
    long long* cv = ct.cnt + g * 2 * kMaxCtx;
    if (chain_start) {
      for (int c = 0; c < NCTX; c++) cv[kMaxCtx + c] = tot[c];
      publish(ct, g, 0, 2);
    } else {
      for (int c = 0; c < NCTX; c++) cv[c] = tot[c];
      publish(ct, g, 0, 1);
      long long j = g - 1;
      long long jmin = g - tin;
      for (;;) {
        int st = wait_state(ct, j, 0, status);
        volatile const long long* pv = ct.cnt + j * 2 * kMaxCtx;
        if (st == 2) {
          for (int c = 0; c < NCTX; c++) incnt[c] += pv[kMaxCtx + c];
          break;
        }
        for (int c = 0; c < NCTX; c++) incnt[c] += pv[c];
        if (st == 0 || j == jmin) break;
        j--;
      }
      for (int c = 0; c < NCTX; c++) cv[kMaxCtx + c] = incnt[c] + tot[c];
      publish(ct, g, 0, 2);
    }
  }
#pragma unroll
  for (int c = 0; c < NCTX; c++) incnt[c] = __shfl_sync(0xffffffffu, incnt[c], 0);

  // ---- 2. A-maps ----
  AMap m[NCTX];
  long long idx[NCTX];
#pragma unroll
  for (int c = 0; c < NCTX; c++) {
    m[c] = amap_identity();
    idx[c] = incnt[c] + lbase[c];
  }
  gen.for_each([&](int ctx, int v, int xl, uint32_t xb) {
    m[ctx] = amap_push(m[ctx], v, halves_after(idx[ctx]));
    idx[ctx]++;
  });
  AMap pre[NCTX], agg[NCTX];
#pragma unroll
  for (int c = 0; c < NCTX; c++) pre[c] = warp_excl_amap(m[c], &agg[c]);
  int ain[NCTX];
  if (lane == 0) {
    int* sv = ct.states + g * kMaxCtx;
    for (int c = 0; c < NCTX; c++) ain[c] = 4;  // AdaptiveRiceState: A = 4, N = 1
    if (!chain_start) {
      AMap* mv = ct.maps + g * kMaxCtx;
      for (int c = 0; c < NCTX; c++) mv[c] = agg[c];
      publish(ct, g, 1, 1);
      AMap acc[NCTX];
      for (int c = 0; c < NCTX; c++) acc[c] = amap_identity();
      long long j = g - 1;
      long long jmin = g - tin;
      for (;;) {
        int st = wait_state(ct, j, 1, status);
        if (st == 2) {
          volatile const int* ps = ct.states + j * kMaxCtx;
          for (int c = 0; c < NCTX; c++) ain[c] = (int)amap_apply(acc[c], ps[c]);
          break;
        }
        volatile const AMap* pm = ct.maps + j * kMaxCtx;
        for (int c = 0; c < NCTX; c++) {
          AMap a;
          a.c = pm[c].c;
          a.s = pm[c].s;
          a.t = pm[c].t;
          acc[c] = amap_then(a, acc[c]);
        }
        if (st == 0 || j == jmin) {
          for (int c = 0; c < NCTX; c++) ain[c] = (int)amap_apply(acc[c], 4);
          break;
        }
        j--;
      }
    }
    for (int c = 0; c < NCTX; c++) sv[c] = (int)amap_apply(agg[c], ain[c]);
    publish(ct, g, 1, 2);
  }
  long long A[NCTX];
#pragma unroll
  for (int c = 0; c < NCTX; c++) {
    ain[c] = __shfl_sync(0xffffffffu, ain[c], 0);
    A[c] = amap_apply(pre[c], ain[c]);
    idx[c] = incnt[c] + lbase[c];
  }

  // ---- 3. code lengths ----
  long long nbits = 0;
  {
    long long A2[NCTX], i2[NCTX];
#pragma unroll
    for (int c = 0; c < NCTX; c++) A2[c] = A[c], i2[c] = idx[c];
    gen.for_each([&](int ctx, int v, int xl, uint32_t xb) {
      int k = select_k(A2[ctx], n_before(i2[ctx]));
      nbits += rice_len(v, k) + xl;
      A2[ctx] = (A2[ctx] + v) >> halves_after(i2[ctx]);
      i2[ctx]++;
    });
  }
  long long tbits;
  long long loff = warp_excl_sum(nbits, &tbits);
  long long toff = 0;
  if (lane == 0) {
    unsigned long long* bv = ct.bitv + g * 2;
    if (chain_start) {
      bv[0] = (unsigned long long)tbits;
      bv[1] = (unsigned long long)tbits;
      publish(ct, g, 2, 2);
    } else {
      bv[0] = (unsigned long long)tbits;
      publish(ct, g, 2, 1);
      long long j = g - 1, jmin = g - tin;
      for (;;) {
        int st = wait_state(ct, j, 2, status);
        volatile const unsigned long long* pv = ct.bitv + j * 2;
        if (st == 2) {
          toff += (long long)pv[1];
          break;
        }
        toff += (long long)pv[0];
        if (st == 0 || j == jmin) break;
        j--;
      }
      bv[1] = (unsigned long long)(toff + tbits);
      publish(ct, g, 2, 2);
    }
    long long ntile_chain = ct.tile_base[chain + 1] - ct.tile_base[chain];
    if (tin == ntile_chain - 1) ct.bits[chain] = (unsigned long long)(toff + tbits);
  }
  toff = __shfl_sync(0xffffffffu, toff, 0);

  // ---- 4. emit ----
  WordSink sink;
  sink.words = reinterpret_cast<uint32_t*>(ct.out[chain]);
  sink.cap_words = ct.cap[chain] / 4;
  sink.tile_first_word = toff >> 5;
  sink.tile_start_partial = (toff & 31) != 0;
  sink.edge = ct.edge + g * 2;
  sink.status = status;
  const long long s_l = toff + loff, e_l = s_l + nbits;
  LaneBits lb;
  lb.init(s_l, &sink);
  gen.for_each([&](int ctx, int v, int xl, uint32_t xb) {
    int k = select_k(A[ctx], n_before(idx[ctx]));
    lb.put(rice_bits(v, k), rice_len(v, k));
    if (xl) {
      if (xl > 16) {
        lb.put(xb >> 16, xl - 16);
        lb.put(xb & 0xFFFFu, 16);
      } else {
        lb.put(xb, xl);
      }
    }
    A[ctx] = (A[ctx] + v) >> halves_after(idx[ctx]);
    idx[ctx]++;
  });
  // lane partial words: head (word s_l>>5, started mid-word) and/or tail (bits left in acc)
  const bool has_tail = lb.nacc > 0 && nbits > 0;
  uint32_t tail = has_tail ? (uint32_t)(lb.acc << (32 - lb.nacc)) : 0u;
  const long long tail_word = lb.wpos;
  // single: the lane's bits sit inside one word that it does not complete
  const bool single = nbits > 0 && has_tail && tail_word == lb.first && lb.head_partial;
  // carry loop over lanes, in order
  long long cw = -1;
  uint32_t cb = 0;
  for (int l = 0; l < 32; l++) {
    long long ncw = cw;
    uint32_t ncb = cb;
    if (lane == l && nbits > 0) {
      if (single) {
        uint32_t w = (cw == lb.first ? cb : 0u) | tail;
        ncw = lb.first;
        ncb = w;
      } else {
        if (lb.have_head) {
          uint32_t w = (cw == lb.first ? cb : 0u) | lb.head;
          sink.write(lb.first, w);
        }
        if (has_tail) {
          ncw = tail_word;
          ncb = tail;
        } else {
          ncw = -1;
          ncb = 0;
        }
      }
    }
    cw = __shfl_sync(0xffffffffu, ncw, l);
    cb = __shfl_sync(0xffffffffu, ncb, l);
  }
  // the tile's last partial word: parked for the fix-up pass (a later tile may add bits)
  if (lane == 0 && cw >= 0) {
    if (cw == sink.tile_first_word && sink.tile_start_partial) sink.edge[0] = cb;
    else sink.edge[1] = cb;
  }
  (void)e_l;
}

// ---------------------------------------------------------------------------
// Plane coder tile = one row (encode_plane, _kernels.py:169-216)
// ---------------------------------------------------------------------------
enum { kFree = 0, kForced = 1, kInRun = 2 };

struct PlaneRow {
  const uint8_t* cur;
  const uint8_t* prev;  // nullptr on row 0
  int w;
  int x0, x1;           // lane slice
  int entry;            // automaton state entering the slice
  long long cont_next;  // run continuation entering the next lane

  // _neighbors, _kernels.py:131-143
  __device__ __forceinline__ void abc(int x, int& a, int& b, int& c) const {
    a = x > 0 ? cur[x - 1] : (prev ? prev[x] : 128);
    b = prev ? prev[x] : a;
    c = (x > 0 && prev) ? prev[x - 1] : b;
  }
  __device__ __forceinline__ bool ebit(int x) const {
    int a, b, c;
    abc(x, a, b, c);
    return cur[x] == a;
  }

  template <class Fn>
  __device__ __forceinline__ void for_each(Fn&& f) const {
    int st = entry;
    for (int x = x0; x < x1; x++) {
      int a, b, c;
      abc(x, a, b, c);
      const int xv = cur[x];
      const bool E = xv == a;
      if (st == kFree && a == b && b == c) {
        // run mode: run = samples equal to a from x; chunks of <= 255, 255 continues
        long long L = 0;
        int xx = x;
        bool e = E;
        while (e) {
          L++;
          xx++;
          if (xx >= x1) break;
          e = cur[xx] == cur[xx - 1];
        }
        if (xx >= x1 && e) L += cont_next;
        long long rem = L;
        for (;;) {
          int ch = rem >= 255 ? 255 : (int)rem;
          f(kRunCtx, ch, 0, 0u);
          rem -= ch;
          if (ch < 255) break;
        }
        st = kInRun;
      }
      if (st == kInRun) {
        if (E) continue;
        st = kForced;
      }
      // regular sample: MED prediction, activity context, folded residual
      int mx = max(a, b), mn = min(a, b);
      int pred = c >= mx ? mn : (c <= mn ? mx : a + b - c);
      int g = abs(a - c) + abs(c - b);
      int ctx = g == 0 ? 0 : (g <= 2 ? 1 : (g <= 8 ? 2 : 3));
      int r = (xv - pred) & 255;
      if (r > 127) r -= 256;
      int u = r >= 0 ? 2 * r : -2 * r - 1;
      f(ctx, u, 0, 0u);
      st = kFree;
    }
  }
};

__device__ __forceinline__ int slice_transition(const PlaneRow& pr, int st0) {
  int st = st0;
  for (int x = pr.x0; x < pr.x1; x++) {
    int a, b, c;
    pr.abc(x, a, b, c);
    bool E = pr.cur[x] == a;
    if (st == kFree && a == b && b == c) st = kInRun;
    if (st == kInRun) {
      if (E) continue;
      st = kForced;
    }
    st = kFree;
  }
  return st;
}

// ---------------------------------------------------------------------------
// DCT coder tile = 32 blocks of one component (encode_dct_component)
// ---------------------------------------------------------------------------
struct DctBlock {
  const int16_t* z;  // this block's 64 zigzag coefficients (nullptr: lane idle)
  int prev_dc;
  int base;          // context bank: 0 luma, 3 chroma

  __device__ __forceinline__ static int bitlen(unsigned u) { return u ? 32 - __clz(u) : 0; }
  __device__ __forceinline__ static unsigned interleave(int v) { return v >= 0 ? 2u * v : (unsigned)(-2 * v - 1); }

  template <class Fn>
  __device__ __forceinline__ void for_each(Fn&& f) const {
    if (!z) return;
    int dc = z[0];
    unsigned u = interleave(dc - prev_dc);
    int s = bitlen(u);
    f(base, s, s, u);
    int pos = 1;
    while (pos < 64) {
      int nz = -1;
      for (int j = pos; j < 64; j++)
        if (z[j] != 0) {
          nz = j;
          break;
        }
      if (nz < 0) {
        f(base + 1, kEOB, 0, 0u);
        break;
      }
      f(base + 1, nz - pos, 0, 0u);
      u = interleave(z[nz]);
      s = bitlen(u);
      f(base + 2, s, s, u);
      pos = nz + 1;
    }
  }
};

// ---------------------------------------------------------------------------
// Kernels: a warp takes the next ticket = next global tile.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_chain(const ChainTab& ct, long long g) {  // chain of global tile g
  int lo = 0, hi = ct.nchains;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (ct.tile_base[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(128) k_entropy(const ImgDesc* __restrict__ descs, ChainTab ct) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    long long t = 0;
    if (lane == 0) t = atomicAdd(ct.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ct.ntiles) return;
    // round-robin over chains: all chains advance together, every wait is on an older ticket
    int k = 0;
    while (k + 1 < ct.nseg && ct.seg_t0[k + 1] <= t) k++;
    const long long rel = t - ct.seg_t0[k];
    const int act = ct.seg_active[k];
    const long long tin = ct.seg_r0[k] + rel / act;
    const int chain = ct.rr_chain[rel % act];
    const long long g = ct.tile_base[chain] + tin;
    const ImgDesc& d = descs[ct.img[chain]];
    const int kind = ct.kind[chain];
    if (kind == 0) {
      const long long tpc = (d.nblocks + 31) / 32;
      const int ci = (int)(tin / tpc);
      const long long bi = (tin % tpc) * 32 + lane;
      DctBlock blk;
      blk.base = ci == 0 ? 0 : 3;
      blk.z = nullptr;
      blk.prev_dc = 0;
      if (bi < d.nblocks) {
        blk.z = d.zz + ((long long)ci * d.nblocks + bi) * 64;
        blk.prev_dc = bi > 0 ? d.zz[((long long)ci * d.nblocks + bi - 1) * 64] : 0;
      }
      run_tile<6>(ct, chain, tin, g, blk, d.status);
    } else {
      const int y = (int)tin;
      const uint8_t* src = kind == 1 ? d.e_plane : d.res_planes + (long long)(kind - 2) * d.n;
      PlaneRow pr;
      pr.cur = src + (long long)y * d.w;
      pr.prev = y > 0 ? src + (long long)(y - 1) * d.w : nullptr;
      pr.w = d.w;
      const int P = (d.w + 31) / 32;
      pr.x0 = min(d.w, lane * P);
      pr.x1 = min(d.w, pr.x0 + P);
      // slice transition functions for the 3 entry states, composed across lanes
      int T = slice_transition(pr, kFree) | (slice_transition(pr, kForced) << 2) |
              (slice_transition(pr, kInRun) << 4);
      int comp = T;  // inclusive composition (apply lower lanes first)
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, comp, dd);
        if (lane >= dd) {
          int r = 0;
          for (int s = 0; s < 3; s++) r |= ((comp >> (2 * ((o >> (2 * s)) & 3))) & 3) << (2 * s);
          comp = r;
        }
      }
      int excl = __shfl_up_sync(0xffffffffu, comp, 1);
      pr.entry = lane == 0 ? kFree : (excl & 3);  // prefix applied to kFree
      // leading run continuation: lead = E-ones from the slice start, pass = whole slice
      long long lead = 0;
      for (int x = pr.x0; x < pr.x1 && pr.ebit(x); x++) lead++;
      bool pass = lead == pr.x1 - pr.x0;
      long long val = lead;
      bool fl = pass;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        long long ov = __shfl_down_sync(0xffffffffu, val, dd);
        bool of = __shfl_down_sync(0xffffffffu, fl, dd);
        if (lane + dd < 32) {
          if (fl) {
            val += ov;
            fl = of;
          }
        } else {
          fl = false;
        }
      }
      long long nx = __shfl_down_sync(0xffffffffu, val, 1);
      pr.cont_next = lane == 31 ? 0 : nx;
      run_tile<5>(ct, chain, tin, g, pr, d.status);
    }
  }
}

// Merge the words shared between tiles.  Word w belongs to the tile holding
// its first bit; that tile's tail plus the heads of the following tiles that
// start inside w (several, if tiles are tiny) are OR-ed and stored once.
__global__ void __launch_bounds__(256) k_entropy_fixup(ChainTab ct) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ct.ntiles) return;
  const int chain = find_chain(ct, g);
  const long long gend = ct.tile_base[chain + 1];
  const long long e = (long long)ct.bitv[g * 2 + 1];
  const long long s = e - (long long)ct.bitv[g * 2 + 0];
  if (e == s || (e & 31) == 0) return;
  const long long w = (e - 1) >> 5;
  if ((s >> 5) == w && (s & 31) != 0) return;  // starts inside w: not the owner
  uint32_t v = ct.edge[g * 2 + 1];
  for (long long j = g + 1; j < gend; j++) {
    const long long ej = (long long)ct.bitv[j * 2 + 1];
    const long long sj = ej - (long long)ct.bitv[j * 2 + 0];
    if (sj >= ((w + 1) << 5)) break;
    if (ej > sj) v |= ct.edge[j * 2 + 0];
    if (ej >= ((w + 1) << 5)) break;
  }
  uint32_t* words = reinterpret_cast<uint32_t*>(ct.out[chain]);
  if (w < ct.cap[chain] / 4) words[w] = __byte_perm(v, 0, 0x0123);
}

void launch_entropy_fixup(const ChainTab& ct, cudaStream_t st) {
  k_entropy_fixup<<<(unsigned)((ct.ntiles + 255) / 256), 256, 0, st>>>(ct);
}

void launch_entropy(const ImgDesc* d_descs, const ChainTab& ct, cudaStream_t st) {
  int warps_per_block = 4;
  long long blocks = (ct.ntiles + warps_per_block - 1) / warps_per_block;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_entropy<<<(unsigned)blocks, 32 * warps_per_block, 0, st>>>(d_descs, ct);
}

}  // namespace hdll
