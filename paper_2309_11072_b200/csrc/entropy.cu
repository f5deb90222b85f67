// entropy.cu -- the two adaptive Golomb-Rice coders, parallelised.
//
// Reference (sequential, numba):
//   encode_plane          _kernels.py:169-216  (lossless coder id 1: MED + 5 contexts + runs)
//   encode_dct_component  _kernels.py:280-324  (base layer symbols, 6 contexts; Y uses 0-2,
//                                               Cb and Cr share 3-5, codec_core.py:439-450)
//   _rice_put / _select_k / _update_state      _kernels.py:65-128
//
// Parallel form.  A *chain* is one sequential coder invocation (one DCT stream
// per image, one plane stream per (image, plane)); it is cut into *tiles*
// (32 plane rows, or 32 consecutive DCT blocks of one component), one warp per
// tile, lane = one row / one block: a contiguous range of the chain's symbols.
// The symbols of a tile depend only on the data; the coder state carried
// between tiles is, per context, (count, A).  Each warp derives its lanes'
// symbols from the data (once per pass) and runs three chained decoupled
// look-backs (tickets are dealt round-robin over the chains in order, so every
// wait is on an older, running warp):
//   1. counts per context  -> global symbol index (halving points, N)
//   2. A-maps per context  -> incoming A of the tile (common.cuh AMap)
//   3. code lengths        -> bit offset of the tile in its chain
//   4. emit MSB-first bits straight into the chain's byte stream; words shared
//      between lanes merge through a warp carry, the (at most two) words a
//      tile shares with its neighbours are parked in `edge` and merged by
//      k_entropy_fixup, so no warp ever waits on another's emission.
// Flags carry the launch epoch, so status memory is never re-zeroed.
#include <algorithm>

#include "encoder.cuh"

namespace hdll {

// A tile whose predecessor has not published yet sleeps between polls: the
// spinning warps otherwise take issue slots from the ones doing the coding
// (3 us measured best: config 1 -0.38 ms against 20 ns; 10 us and backoff
// were slower).  A predecessor is always in flight, so waits are bounded by
// one tile's work; kSpinLimit polls (seconds) only guard against a bug.
#ifndef HDLL_LB_SLEEP_NS
#define HDLL_LB_SLEEP_NS 3000
#endif
constexpr unsigned kLookbackSleepNs = HDLL_LB_SLEEP_NS;
constexpr long long kSpinLimit = 1LL << 20;

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
// smallest k <= 15 with (N << k) >= A  (_select_k, _kernels.py:114-119), closed form
__device__ __forceinline__ int kfast(int a, int n) {
  if (a <= n) return 0;
  int k0 = __clz(n) - __clz(a - 1);  // bitlen(a-1) - bitlen(n) >= 0
  int k = ((n << k0) >= a) ? k0 : k0 + 1;
  return k < kRiceMaxK ? k : kRiceMaxK;
}

// kfast without the a <= n branch: bitlen(a - 1) - bitlen(n), clamped at 0,
// plus one when n << k0 still falls short of a
__device__ __forceinline__ int kfast_bf(int a, int n) {
  int k0 = max(__clz(n) - __clz(max(a - 1, 0)), 0);
  k0 += (n << k0) < a ? 1 : 0;
  return min(k0, kRiceMaxK);
}

__device__ __noinline__ AMap amap_push_slow(AMap m, int u, int h) { return amap_push(m, u, h); }
__device__ __noinline__ AMap amap_then_call(AMap f, AMap g) { return amap_then(f, g); }
// exact o exact with a small total shift is the common case: inline it
__device__ __forceinline__ AMap amap_then_slow(const AMap& f, const AMap& g) {
  if (f.s >= 0 && g.s >= 0 && f.s + g.s < kADomainBits && f.s < 20) {
    AMap r;
    r.c = f.c + (g.c << f.s);
    r.s = f.s + g.s;
    r.t = 0;
    return r;
  }
  return amap_then_call(f, g);
}

// the plane coder's packed map state (run_tile) past the exact range: through AMap
__device__ __noinline__ void plane_map_push_slow(int* x, int* c, int* t, int u, int h) {
  const int n = *x & 63, sft = *x >> 8;
  AMap m = sft == 15 ? AMap{*c, -1, *t} : AMap{*c, sft, 0};
  m = amap_push(m, u, h);
  const int nn = h ? kStateReset / 2 : n + 1;
  *x = nn | ((m.s < 0 ? 15 : m.s) << 8);
  *c = (int)m.c;
  *t = m.t;
}

__device__ __forceinline__ void amap_push_fast(AMap& m, int u, int h) {
  if (m.s >= 0 && m.s + h < kADomainBits) {
    m.c += (long long)u << m.s;
    m.s += h;
  } else {
    m = amap_push_slow(m, u, h);
  }
}

__device__ __forceinline__ AMap warp_excl_amap_small(const AMap& m, AMap* total) {
  const unsigned lane = threadIdx.x & 31u;
  AMap x = m;
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {
    AMap y = shfl_up_amap(x, d);
    if (lane >= (unsigned)d) x = amap_then_slow(y, x);
  }
  *total = shfl_amap(x, 31);
  AMap ex = shfl_up_amap(x, 1);
  if (lane == 0) ex = amap_identity();
  return ex;
}

__device__ __forceinline__ int wait_state(const ChainTab& ct, long long g, int which, unsigned* status) {
  const int* f = ct.flags + g * 4 + which;
  for (long long it = 0;; it++) {
    int v = ld_acquire(f);
    if ((v >> 2) == ct.epoch && (v & 3)) return v & 3;
    if (it > kSpinLimit) {
      atomicOr(status, kErrLookback);
      return 0;
    }
    __nanosleep(kLookbackSleepNs);
  }
}

__device__ __forceinline__ void publish(const ChainTab& ct, long long g, int which, int state) {
  st_release(ct.flags + g * 4 + which, (ct.epoch << 2) | state);
}

// Warp-parallel look-back: lane l probes predecessor tile j0 - l (>= jmin).
// Waits until every valid tile of the window has published phase `which`;
// returns the lowest lane holding an inclusive prefix (32 if none) and the
// lane's own state (0 outside the chain, 1 aggregate, 2 inclusive).
__device__ __forceinline__ int probe_window(const ChainTab& ct, long long j0, long long jmin, int which,
                                            unsigned* status, int* my_state) {
  const int lane = threadIdx.x & 31;
  const long long j = j0 - lane;
  const bool valid = j >= jmin;
  const int* f = ct.flags + (valid ? j : 0) * 4 + which;
  int st = 0;
  for (long long it = 0;; it++) {
    if (valid && st == 0) {
      const int v = ld_acquire(f);
      if ((v >> 2) == ct.epoch && (v & 3)) st = v & 3;
    }
    if (__all_sync(0xffffffffu, !valid || st != 0)) break;
    if (it > kSpinLimit) {
      if (lane == 0) atomicOr(status, kErrLookback);
      if (valid && st == 0) st = 2;  // give up: treat as a (garbage) prefix, never hang
      break;
    }
    __nanosleep(kLookbackSleepNs);
  }
  *my_state = valid ? st : 0;
  const unsigned incl = __ballot_sync(0xffffffffu, valid && st == 2);
  return incl ? __ffs(incl) - 1 : 32;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// composition of the lanes' maps, oldest (highest lane) first; result in every lane
__device__ __forceinline__ AMap warp_compose_down(AMap x) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {
    AMap y;
    y.c = __shfl_down_sync(0xffffffffu, x.c, d);
    y.s = __shfl_down_sync(0xffffffffu, x.s, d);
    y.t = __shfl_down_sync(0xffffffffu, x.t, d);
    if (lane + d < 32) x = amap_then_slow(y, x);
  }
  return shfl_amap(x, 0);
}

// ticket -> (chain, tile-in-chain, global tile) through the round-robin schedule
// kCM: the launch carries per-chain modes (row-band pieces, band.cu).  The
// whole-image encode compiles without them: a per-tile mode lookup in the
// coding kernels measured +0.34 ms on config 1 (A/B, profiles/r02).
template <bool kCM>
__device__ __forceinline__ int chain_mode(const ChainTab& ct, int chain) {
  if constexpr (kCM) return ct.chain_mode[chain];
  return ct.mode;
}

// the next ticket's tile, passing over the tiles of chains that are not run
template <bool kCM>
__device__ __forceinline__ bool next_tile(const ChainTab& ct, int* chain, long long* tin, long long* g) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    long long t = 0;
    if (lane == 0) t = atomicAdd(ct.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ct.ntiles) return false;
    int k = 0;
    while (k + 1 < ct.nseg && ct.seg_t0[k + 1] <= t) k++;
    const long long rel = t - ct.seg_t0[k];
    const int act = ct.seg_active[k];
    *tin = ct.seg_r0[k] + rel / act;
    *chain = ct.rr_chain[rel % act];
    *g = ct.tile_base[*chain] + *tin;
    if (!kCM || chain_mode<kCM>(ct, *chain) != kModeSkip) return true;
  }
}

// ---------------------------------------------------------------------------
// Bit emission
// ---------------------------------------------------------------------------
struct WordSink {
  uint32_t* words;
  long long cap_words;
  long long tile_first_word;
  bool tile_start_partial;
  uint32_t* edge;  // this tile's [head, tail] slots
  unsigned* status;

  __device__ __forceinline__ void write(long long idx, uint32_t w) const {
    if (idx == tile_first_word && tile_start_partial) {
      edge[0] = w;  // shared with the previous tile: merged by the fix-up pass
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
  unsigned long long acc;
  int nacc;
  long long wpos, first;
  bool head_partial, have_head;
  uint32_t head;

  __device__ __forceinline__ void init(long long s) {
    wpos = first = s >> 5;
    nacc = (int)(s & 31);
    acc = 0;
    head_partial = nacc != 0;
    have_head = false;
  }
  __device__ __forceinline__ void put(const WordSink& sink, uint32_t bits, int len) {
    acc = (acc << len) | (unsigned long long)bits;
    nacc += len;
    if (nacc >= 32) {
      uint32_t w = (uint32_t)(acc >> (nacc - 32));
      nacc -= 32;
      acc &= (1ULL << nacc) - 1ULL;
      if (wpos == first && head_partial) {
        head = w;
        have_head = true;
      } else {
        sink.write(wpos, w);
      }
      wpos++;
    }
  }
};

// A lane's code bits before its position in the stream is known: MSB-first
// 32-bit words at w[j * 32] (lanes interleaved), copied into place by the emit
// pass once the look-back has given the lane its bit offset.
struct ScratchBits {
  uint32_t* w;
  int cap, n, nacc;
  unsigned long long acc;
  __device__ __forceinline__ void init(uint32_t* p, int c) {
    w = p;
    cap = c;
    n = nacc = 0;
    acc = 0;
  }
  __device__ __forceinline__ void put(uint32_t bits, int len) {  // len <= 32
    acc = (acc << len) | (unsigned long long)bits;
    nacc += len;
    if (nacc >= 32) {
      nacc -= 32;
      if (n < cap) w[n * 32] = (uint32_t)(acc >> nacc);
      n++;
    }
  }
  __device__ __forceinline__ void flush() {
    if (nacc) {
      if (n < cap) w[n * 32] = (uint32_t)(acc << (32 - nacc));
      n++;
      nacc = 0;
    }
  }
};

// ---------------------------------------------------------------------------
// Symbol sources.  A generator enumerates a lane's symbols in coder order as
// f(index, ctx, value, raw_len, raw_bits), re-deriving them from the data on
// every pass (DCT blocks below, plane rows further down).
// ---------------------------------------------------------------------------
// One 8x8 block of zigzag coefficients (encode_dct_component, _kernels.py:280-324):
// DC size (ctx 0) + raw bits, then per nonzero AC (zero run ctx 1, size ctx 2 +
// raw bits), EOB = run 64 unless position 63 is coded.
struct DctBlockGen {
  static constexpr bool kStaticCtx = true;  // every f() call names its context
  const int16_t* z;  // nullptr: idle lane
  unsigned long long nzm;
  unsigned dcu;      // interleaved DC difference
  template <class F>
  __device__ __forceinline__ void for_each(F&& f) const {
    if (!z) return;
    int s = dcu ? 32 - __clz(dcu) : 0;
    f(0, 0, s, s, dcu);
    // (loading the next nonzero's coefficient one symbol ahead measured
    // slower: entropy_dct 2.85 -> 2.95 ms on config 1)
    int pos = 1, i = 1;
    while (pos < 64) {
      const unsigned long long rest = nzm >> pos;
      if (rest == 0) {
        f(i, 1, kEOB, 0, 0u);
        break;
      }
      const int nz = pos + __ffsll((long long)rest) - 1;
      f(i++, 1, nz - pos, 0, 0u);
      const int zv = __ldg(z + nz);
      const unsigned u = zv >= 0 ? 2u * zv : (unsigned)(-2 * zv - 1);
      s = 32 - __clz(u);
      f(i++, 2, s, s, u);
      pos = nz + 1;
    }
  }
};

// A lane's run of consecutive blocks (their nonzero masks and DC differences
// staged in shared memory by the count pass): the blocks' symbols in order.
struct DctRunGen {
  static constexpr bool kStaticCtx = true;
  const int16_t* z0;                    // the first block's coefficients (nullptr: idle lane)
  const unsigned long long* nzm;        // [k * 32] this lane's masks, stride 32
  const unsigned* dcu;                  // [k * 32]
  int nb;                               // blocks of the lane
  template <class F>
  __device__ __forceinline__ void for_each(F&& f) const {
    if (!z0) return;
    int i = 0;
    for (int k = 0; k < nb; k++) {
      DctBlockGen b{z0 + 64LL * k, nzm[32 * k], dcu[32 * k]};
      b.for_each([&](int, int c, int v, int xl, uint32_t xb) { f(i++, c, v, xl, xb); });
    }
  }
};

// Per-lane context state lives in shared memory, [context][lane], so a symbol
// touches only its own context (no per-context predication).
struct LaneState {
  long long* mc;  // map constant
  int* ms;        // map shift (< 0: step map)
  int* mt;        // step-map threshold
  int* a;         // A
  int* nn;        // N
};

// ---------------------------------------------------------------------------
// The tile engine over a lane's symbol list in shared memory.
//   NL local contexts used by the tile, mapped to chain contexts base..base+NL-1,
//   NC contexts carried by the chain.
// ---------------------------------------------------------------------------
template <int NL, int NC, bool kCM, class Gen>
__device__ void run_tile(const ChainTab& ct, int chain, long long tin, long long g, int base, const Gen& gen,
                         const int* cnt_in, const LaneState& ls, unsigned* status, uint32_t* scr, int scr_cap) {
  const int lane = threadIdx.x & 31;
  const int mode = chain_mode<kCM>(ct, chain);
#ifdef HDLL_EXP_NO_LB  // timing experiment only: no look-backs (wrong output)
  const bool chain_start = true;
#else
  const bool chain_start = tin == 0;
#endif

  // ---- 1. counts -> global symbol index of this lane's first symbol per context ----
  long long lbase[NL], tot[NL];
#pragma unroll
  for (int c = 0; c < NL; c++) {
    long long t;
    lbase[c] = warp_excl_sum((long long)cnt_in[c], &t);
    tot[c] = t;
  }
  const bool chain_last = tin == ct.tile_base[chain + 1] - ct.tile_base[chain] - 1;
  long long incnt[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) incnt[c] = chain_start ? ct.in_cnt[chain * kMaxCtx + c] : 0;
  if (!chain_start) {
    if (lane == 0) {
      long long* cv = ct.cnt + g * 2 * kMaxCtx;
#pragma unroll
      for (int c = 0; c < NC; c++) cv[c] = (c >= base && c < base + NL) ? tot[c - base] : 0;
      publish(ct, g, 0, 1);
    }
    const long long jmin = g - tin;
    for (long long j0 = g - 1;; j0 -= 32) {
      int st;
      const int k = probe_window(ct, j0, jmin, 0, status, &st);
      const long long j = j0 - lane;
      volatile const long long* pv = ct.cnt + (st ? j : 0) * 2 * kMaxCtx;
#pragma unroll
      for (int c = 0; c < NC; c++) {
        long long v = 0;
        if (st && lane < k) v = pv[c];
        else if (st && lane == k) v = pv[kMaxCtx + c];
        incnt[c] += warp_sum_ll(v);
      }
      if (k < 32) break;
    }
  }
  if (lane == 0) {
    long long* cv = ct.cnt + g * 2 * kMaxCtx;
#pragma unroll
    for (int c = 0; c < NC; c++) cv[kMaxCtx + c] = incnt[c] + ((c >= base && c < base + NL) ? tot[c - base] : 0);
    publish(ct, g, 0, 2);
    if (mode != 2 && chain_last)
      for (int c = 0; c < NC; c++) ct.out_cnt[chain * kMaxCtx + c] = cv[kMaxCtx + c];
  }
  if (mode == 1) return;
  int n0[NL];  // N before this lane's first symbol of each context
#pragma unroll
  for (int c = 0; c < NL; c++) n0[c] = n_before(incnt[base + c] + lbase[c]);

  // ---- 2. A-maps (the reference's update_state as a map of the incoming A) ----
#pragma unroll
  for (int c = 0; c < NL; c++) {
    ls.mc[c * 32 + lane] = 0;
    ls.ms[c * 32 + lane] = 0;
    ls.mt[c * 32 + lane] = 0;
    ls.nn[c * 32 + lane] = n0[c];
  }
#ifndef HDLL_EXP_NO_MAPS
  if constexpr (Gen::kStaticCtx) {  // every call site names its context: the state stays in registers
    long long rmc[NL];
    int rms[NL], rmt[NL], rnn[NL];
#pragma unroll
    for (int c = 0; c < NL; c++) rmc[c] = 0, rms[c] = 0, rmt[c] = 0, rnn[c] = n0[c];
    gen.for_each([&](int, int c, int v, int, uint32_t) {
      const int nb = rnn[c];
      const int h = nb == kStateReset - 1;  // N reaches 64: A and N halve
      rnn[c] = h ? kStateReset / 2 : nb + 1;
      const int sft = rms[c];
      if (sft >= 0 && sft + h < kADomainBits) {
        rmc[c] += (long long)v << sft;
        rms[c] = sft + h;
      } else {
        AMap m{rmc[c], sft, rmt[c]};
        m = amap_push_slow(m, v, h);
        rmc[c] = m.c;
        rms[c] = m.s;
        rmt[c] = m.t;
      }
    });
#pragma unroll
    for (int c = 0; c < NL; c++) {
      ls.mc[c * 32 + lane] = rmc[c];
      ls.ms[c * 32 + lane] = rms[c];
      ls.mt[c * 32 + lane] = rmt[c];
    }
  } else {
    // Per context one shared word X = N | shift << 8 (shift 15: a step map)
    // and the map constant in 32 bits: while exact (shift < 14) it stays below
    // 255 * (63 + 32 * (2^14 - 2)) < 2^28.
    int* X = ls.nn;
    int* C = ls.a;
#pragma unroll
    for (int c = 0; c < NL; c++) C[c * 32 + lane] = 0;
    gen.for_each([&](int, int c, int v, int, uint32_t) {
      const int o = c * 32 + lane;
      const int x = X[o];
      const int h = (x & 63) == kStateReset - 1;  // N reaches 64: A and N halve
      const int xn = x + (h ? 0x100 - (kStateReset / 2 - 1) : 1);
      if (xn < (kADomainBits << 8)) {
        C[o] += v << (x >> 8);
        X[o] = xn;
      } else {
        plane_map_push_slow(X + o, C + o, ls.mt + o, v, h);
      }
    });
#pragma unroll
    for (int c = 0; c < NL; c++) {
      const int o = c * 32 + lane, sft = X[o] >> 8;
      ls.mc[o] = C[o];
      ls.ms[o] = sft == 15 ? -1 : sft;
    }
  }
#endif
  AMap pre[NL], agg[NL];
#pragma unroll 1
  for (int c = 0; c < NL; c++) {
    AMap m{ls.mc[c * 32 + lane], ls.ms[c * 32 + lane], ls.mt[c * 32 + lane]};
    pre[c] = warp_excl_amap_small(m, &agg[c]);
  }
  if (mode == 2) {  // totals only: every tile's aggregate, composed per chain by k_chain_maps
    if (lane == 0) {
      AMap* mv = ct.maps + g * kMaxCtx;
#pragma unroll
      for (int c = 0; c < NC; c++) mv[c] = (c >= base && c < base + NL) ? agg[c - base] : amap_identity();
    }
    return;
  }
  int ain[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) ain[c] = chain_start ? ct.in_a[chain * kMaxCtx + c] : 4;
  if (!chain_start) {
    if (lane == 0) {
      AMap* mv = ct.maps + g * kMaxCtx;
#pragma unroll
      for (int c = 0; c < NC; c++) mv[c] = (c >= base && c < base + NL) ? agg[c - base] : amap_identity();
      publish(ct, g, 1, 1);
    }
    AMap acc[NC];  // composition of the tiles already passed (newer than the window)
#pragma unroll
    for (int c = 0; c < NC; c++) acc[c] = amap_identity();
    const long long jmin = g - tin;
    for (long long j0 = g - 1;; j0 -= 32) {
      int st;
      const int k = probe_window(ct, j0, jmin, 1, status, &st);
      const long long j = j0 - lane;
      volatile const AMap* pm = ct.maps + (st ? j : 0) * kMaxCtx;
      volatile const int* ps = ct.states + (st ? j : 0) * kMaxCtx;
#pragma unroll 1
      for (int c = 0; c < NC; c++) {
        AMap m = amap_identity();
        if (st && lane < k) {
          m.c = pm[c].c;
          m.s = pm[c].s;
          m.t = pm[c].t;
        }
        // a context no tile of the window touched composes to the identity (the
        // DCT chain's Y tiles never touch Cb/Cr's contexts and vice versa)
        if (__any_sync(0xffffffffu, m.c != 0 || m.s != 0))
          acc[c] = amap_then_slow(warp_compose_down(m), acc[c]);
        if (k < 32) ain[c] = (int)amap_apply(acc[c], __shfl_sync(0xffffffffu, st ? ps[c] : 0, k));
      }
      if (k < 32) break;
    }
  }
  if (lane == 0) {
    int* sv = ct.states + g * kMaxCtx;
#pragma unroll
    for (int c = 0; c < NC; c++)
      sv[c] = (c >= base && c < base + NL) ? (int)amap_apply(agg[c - base], ain[c]) : ain[c];
    publish(ct, g, 1, 2);
    if (chain_last)
      for (int c = 0; c < NC; c++) ct.out_a[chain * kMaxCtx + c] = sv[c];
  }

  // ---- 3. codes: every symbol's Rice code (and raw bits) into the lane's scratch words ----
  int a_start[NL];
#pragma unroll
  for (int c = 0; c < NL; c++) {
    a_start[c] = (int)amap_apply(pre[c], ain[base + c]);
    ls.a[c * 32 + lane] = a_start[c];
    ls.nn[c * 32 + lane] = n0[c];
  }
  long long nbits = 0;
  ScratchBits sb;
  sb.init(scr, scr_cap);
  if constexpr (Gen::kStaticCtx) {
    int ra[NL], rnn[NL];
#pragma unroll
    for (int c = 0; c < NL; c++) ra[c] = a_start[c], rnn[c] = n0[c];
    gen.for_each([&](int, int c, int v, int xl, uint32_t xb) {
      const int k = kfast(ra[c], rnn[c]);
      const int rl = rice_len(v, k);
      nbits += rl + xl;
      sb.put(rice_bits(v, k), rl);
      if (xl) sb.put(xb, xl);
      ra[c] += v;  // _update_state
      rnn[c] += 1;
      if (rnn[c] >= kStateReset) {
        ra[c] >>= 1;
        rnn[c] >>= 1;
      }
    });
  } else {
    // (A, N) of a context packed as A | N << 16 in one shared word (A < 2^15)
#pragma unroll
    for (int c = 0; c < NL; c++) ls.a[c * 32 + lane] = a_start[c] | (n0[c] << 16);
    int nb32 = 0;
    gen.for_each([&](int, int c, int v, int xl, uint32_t xb) {  // (plane symbols: v <= 255, no raw bits)
      const int o = c * 32 + lane;
      int st = ls.a[o];
      const int k = kfast_bf(st & 0xFFFF, st >> 16);
      // _rice_put: q ones, a zero, k low bits; q >= 24: 24 ones and 8 raw bits
      const int q = v >> k;
      const bool esc = q >= kRiceEscapeQ;
      const int rl = esc ? kRiceEscapeQ + 8 : q + 1 + k;  // <= 31 unless escaped (v <= 255)
      const uint32_t bits = esc ? (0xFFFFFF00u | (uint32_t)v) : (1u << rl) - ((2u + q) << k) + (uint32_t)v;
      nb32 += rl;
      sb.put(bits, rl);
      st += v + (1 << 16);  // _update_state: A += u, N += 1; at N = 64 both halve
      if (st >= (kStateReset << 16)) st = (st >> 1) & ~0x8000;
      ls.a[o] = st;
    });
    nbits = nb32;
  }
  sb.flush();
  if (sb.n > scr_cap) atomicOr(status, kErrCapacity);
  long long tbits;
  const long long loff = warp_excl_sum(nbits, &tbits);
  long long toff = 0;
  if (lane == 0) {
    ct.bitv[g * 2 + 0] = (unsigned long long)tbits;
    if (!chain_start) publish(ct, g, 2, 1);
  }
  if (!chain_start) {
    const long long jmin = g - tin;
    for (long long j0 = g - 1;; j0 -= 32) {
      int st;
      const int k = probe_window(ct, j0, jmin, 2, status, &st);
      const long long j = j0 - lane;
      volatile const unsigned long long* pv = ct.bitv + (st ? j : 0) * 2;
      long long v = 0;
      if (st && lane < k) v = (long long)pv[0];
      else if (st && lane == k) v = (long long)pv[1];
      toff += warp_sum_ll(v);
      if (k < 32) break;
    }
  }
  if (lane == 0) {
    ct.bitv[g * 2 + 1] = (unsigned long long)(toff + tbits);
    publish(ct, g, 2, 2);
    if (chain_last) ct.bits[chain] = (unsigned long long)(toff + tbits);
  }

  // ---- 4. emit ----
  WordSink sink;
  sink.words = reinterpret_cast<uint32_t*>(ct.out[chain]);
  sink.cap_words = ct.cap[chain] / 4;
  sink.tile_first_word = toff >> 5;
  sink.tile_start_partial = (toff & 31) != 0;
  sink.edge = ct.edge + g * 2;
  sink.status = status;
  LaneBits lb;
  lb.init(toff + loff);
#ifndef HDLL_EXP_NO_EMIT
  {  // the scratch words, shifted into place
    const int nw = min(sb.n, scr_cap);
    int j = 0;
    if constexpr (!Gen::kStaticCtx) {  // plane rows: whole words, four loads in flight before their
      for (; j + 4 < nw; j += 4) {     // stores (-0.17 ms; the DCT's few words per block lose by it)
        uint32_t w4[4];
#pragma unroll
        for (int h = 0; h < 4; h++) w4[h] = scr[(j + h) * 32];
#pragma unroll
        for (int h = 0; h < 4; h++) lb.put(sink, w4[h], 32);
      }
    }
    for (; j < nw; j++) {
      // DCT blocks: the scratch words are read once, evict-first, so the
      // coefficient lines stay in L1 (-0.1 ms; the plane coder loses by it)
      const uint32_t wd = Gen::kStaticCtx ? __ldcs(scr + j * 32) : scr[j * 32];
      const int len = j < nw - 1 ? 32 : (int)(nbits - 32LL * (nw - 1));
      lb.put(sink, len == 32 ? wd : wd >> (32 - len), len);
    }
  }
#endif
  // Lane partial words.  A lane that starts mid-word owes its first word to the
  // carry of the lanes before it; a lane whose bits sit inside one word
  // ("single") passes the carry on OR-ed with its bits.  The carry is a
  // composition of maps x -> x | m (single / empty lanes) and x -> t (lanes
  // ending mid-word), scanned in log2(32) steps.
  const bool has_tail = lb.nacc > 0 && nbits > 0;
  const uint32_t tail = has_tail ? (uint32_t)(lb.acc << (32 - lb.nacc)) : 0u;
  const bool single = has_tail && lb.wpos == lb.first && lb.head_partial;
  // f_l: constant (word, bits) for lanes ending mid-word / aligned (word -1),
  // or x -> x | bits into word `fw` for single lanes, identity (word -2) if empty
  bool c_const = nbits > 0 && !single;
  uint32_t c_val = has_tail ? tail : 0u;
  long long c_word = nbits == 0 ? -2 : (single ? lb.first : (has_tail ? lb.wpos : -1));
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const bool o_const = __shfl_up_sync(0xffffffffu, c_const, dd);
    const uint32_t o_val = __shfl_up_sync(0xffffffffu, c_val, dd);
    const long long o_word = __shfl_up_sync(0xffffffffu, c_word, dd);
    if (lane >= dd && !c_const) {  // compose: earlier (o) then this (c)
      c_val |= o_val;
      c_const = o_const;
      if (c_word == -2) c_word = o_word;
    }
  }
  if (c_word == -2) c_word = -1;  // applied to "no carry"
  // exclusive carry entering this lane
  uint32_t in_val = __shfl_up_sync(0xffffffffu, c_val, 1);
  long long in_word = __shfl_up_sync(0xffffffffu, c_word, 1);
  if (lane == 0) in_val = 0u, in_word = -1;
  if (nbits > 0 && !single && lb.have_head)
    sink.write(lb.first, (in_word == lb.first ? in_val : 0u) | lb.head);
  // the tile's last partial word: parked for the fix-up pass (a later tile may add bits)
  const uint32_t out_val = __shfl_sync(0xffffffffu, c_val, 31);
  const long long out_word = __shfl_sync(0xffffffffu, c_word, 31);
  if (lane == 0 && out_word >= 0) {
    if (out_word == sink.tile_first_word && sink.tile_start_partial) sink.edge[0] = out_val;
    else sink.edge[1] = out_val;
  }
}

// shared-memory bytes of one warp's LaneState for NL contexts
__host__ __device__ constexpr size_t lane_state_bytes(int nl) { return (size_t)nl * 32 * (8 + 4 + 4 + 4 + 4); }

__device__ __forceinline__ LaneState carve_state(uint8_t* p, int nl) {
  LaneState ls;
  ls.mc = reinterpret_cast<long long*>(p);
  ls.ms = reinterpret_cast<int*>(p + (size_t)nl * 32 * 8);
  ls.mt = ls.ms + nl * 32;
  ls.a = ls.mt + nl * 32;
  ls.nn = ls.a + nl * 32;
  return ls;
}

// ---------------------------------------------------------------------------
// Plane coder (encode_plane, _kernels.py:169-216): tile = 32 consecutive rows
// of a plane, lane = one row, so a lane's symbols are one contiguous range of
// the chain and each row starts in the reset automaton state.  The symbols are
// regenerated from the plane (L1-cached loads) by every pass instead of staged.
// ---------------------------------------------------------------------------
// A lane codes one segment [x0, x1) of a row.  Wide rows are cut into S
// segments (plane_segs) so single large images still fill the GPU; a segment
// other than the first enters in the automaton state the previous segments
// leave: either free, or inside a run of L samples so far (the run's chunks
// go out where it ends, _kernels.py:183-198, so no symbol moves between lanes).
// What the coding of a segment entered free tells about entering it inside a
// run: the first sample that differs from its left neighbour (E false) ends any
// run, and both entries code it as a regular sample and leave it outside a run,
// so from there on they emit the same symbols.
struct RowTrack {
  bool brk;    // some sample has E false
  int cov;     // samples before it (all E true)
  int brk_i;   // symbols of the free coding up to and including it
  bool out_in; // exit state of the free coding
  int out_L;
};

// The count pass keeps each row's symbols (u16: ctx << 8 | value)
// in a global scratch slab of the warp, interleaved by lane in 16-byte chunks
// (chunk q of lane l at slab[q * 32 + l]), so the later passes read 8 symbols
// per coalesced 128-bit access instead of re-deriving them.
struct SymChunk {  // 8 u16 symbols, shifted in at the top
  unsigned long long lo = 0, hi = 0;
  __device__ __forceinline__ void push(uint32_t s) {
    lo = (lo >> 16) | (hi << 48);
    hi = (hi >> 16) | ((unsigned long long)s << 48);
  }
  __device__ __forceinline__ uint32_t pop() {  // lowest symbol first
    const uint32_t s = (uint32_t)(lo & 0xFFFFu);
    lo = (lo >> 16) | (hi << 48);
    hi >>= 16;
    return s;
  }
  __device__ __forceinline__ void align(int m) {  // m < 8 pushed: move them to the bottom
    const int sh = 16 * (8 - m);
    if (sh < 64) {
      lo = (lo >> sh) | (hi << (64 - sh));
      hi >>= sh;
    } else {
      lo = hi >> (sh - 64);
      hi = 0;
    }
  }
  __device__ __forceinline__ uint4 word() const {
    return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
  }
  __device__ __forceinline__ void load(const uint4& w) {
    lo = (unsigned long long)w.x | ((unsigned long long)w.y << 32);
    hi = (unsigned long long)w.z | ((unsigned long long)w.w << 32);
  }
};

// The count pass of one segment entered free (_kernels.py:169-216 from a free
// state): every symbol (ctx << 8 | value) into the lane's slab, symbols per
// context, and the RowTrack facts.  _neighbors (_kernels.py:131-143): a = left
// (above at x = 0, 128 at the origin), b = above (else a), c = above-left (else b).
// Samples go four to a 32-bit word with the byte loop unrolled; the regular
// contexts' counts are 8-bit fields of one word, folded out every 16 samples.
// ctx of the activity g = |a - c| + |c - b| (_activity_ctx, _kernels.py:157-166):
// 2-bit fields of kCtxTab indexed by min(g, 9): 0 -> 0, 1-2 -> 1, 3-8 -> 2, 9+ -> 3
constexpr uint32_t kCtxTab = (1u << 2) | (1u << 4) | (2u << 6) | (2u << 8) | (2u << 10) | (2u << 12) | (2u << 14) |
                             (2u << 16) | (3u << 18);

__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t x, uint32_t y) {
  uint32_t r;
  asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
  return r;
}
__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t x, uint32_t y) {
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
  return r;
}

struct SegGen {
  int a, c;           // left and above-left neighbours of the next sample
  bool inrun;
  int L;
  int i;              // symbols so far
  SymChunk ch;
  uint4* sp;          // the slab chunk being filled
  uint32_t cpk;       // regular contexts' counts, 8 bits each (< 256 between folds)
  uint32_t fge2, fge3;  // word4's flags g > 2, g > 8 (16 per flag in a 16-bit lane)
  int nfast;          // word4's regular samples since the last fold
  int cnt[5];
  // RowTrack
  bool brk;
  int cov, brk_i, nsamp;

  __device__ __forceinline__ void put(int ctx, int v) {
    ch.push((uint32_t)((ctx << 8) | v));
    if ((i & 7) == 7) {
      *sp = ch.word();
      sp += 32;
    }
    i++;
  }
  __device__ __forceinline__ void fold() {
    cnt[0] += cpk & 0xFF;
    cnt[1] += (cpk >> 8) & 0xFF;
    cnt[2] += (cpk >> 16) & 0xFF;
    cnt[3] += cpk >> 24;
    cpk = 0;
    const int ge2 = (int)(((fge2 & 0xFFFFu) + (fge2 >> 16)) >> 4), ge3 = (int)(((fge3 & 0xFFFFu) + (fge3 >> 16)) >> 4);
    cnt[1] += nfast - ge2;
    cnt[2] += ge2 - ge3;
    cnt[3] += ge3;
    fge2 = fge3 = 0;
    nfast = 0;
  }
  __device__ __forceinline__ void run_chunks() {  // chunks of <= 255; a chunk of 255 continues
    for (;;) {
      const int chn = L >= 255 ? 255 : L;
      put(kRunCtx, chn);
      cnt[kRunCtx]++;
      L -= chn;
      if (chn < 255) break;
    }
  }
  // one sample (hp: a row above exists; track: record the first break)
  __device__ __forceinline__ void sample(int xv, int braw, bool hp, bool track) {
    const int b = hp ? braw : a;
    const int cc = hp ? c : a;
    const bool E = xv == a;
    if (!inrun && a == b && b == cc) {  // run mode (not forced, a == b == c)
      inrun = true;
      L = 0;
    }
    if (inrun && E) {
      L++;
    } else {
      if (inrun) {  // the run ends: its chunks, then this sample is forced regular
        run_chunks();
        inrun = false;
      }
      // MED = median(a, b, a + b - c) (_med, _kernels.py:146-154), folded residual
      const int mx = max(a, b), mn = min(a, b);
      const int pred = max(mn, min(mx, a + b - cc));
      const int gg = min(abs(a - cc) + abs(cc - b), 9);
      const int ctx = (int)((kCtxTab >> (2 * gg)) & 3u);
      cpk += 1u << (8 * ctx);
      const int t = (xv - pred) << 24;  // r = (x - pred) mod 256 as a signed byte, << 24
      put(ctx, (t >> 23) ^ (t >> 31));   // r >= 0 ? 2r : -2r - 1
    }
    if (track && !E && !brk) {
      brk = true;
      cov = nsamp;
      brk_i = i;
    }
    nsamp++;
    c = b;
    a = xv;
  }
  // four symbols at once (s01: symbols 0, 1; s23: symbols 2, 3, 16 bits each)
  __device__ __forceinline__ void put4(uint32_t s01, uint32_t s23) {
    const unsigned long long S = (unsigned long long)s01 | ((unsigned long long)s23 << 32);
    const int j = i & 7;  // symbols already in the chunk (at its top)
    if (j >= 4) {         // it fills within these four: its 8 symbols start 16 j bits below S
      const int sh = 128 - 16 * j;  // 16..64
      unsigned long long w0, w1;
      if (sh == 64) {
        w0 = ch.hi;
        w1 = S;
      } else {
        w0 = (ch.lo >> sh) | (ch.hi << (64 - sh));
        w1 = (ch.hi >> sh) | (S << (64 - sh));
      }
      *sp = make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32));
      sp += 32;
    }
    ch.lo = ch.hi;
    ch.hi = S;
    i += 4;
  }
  // Four samples (bytes of cw; pw: the row above) of a row with a row above.
  // Outside a run and with no sample whose a == b == c, all four are regular
  // symbols: MED, activity context and folded residual come out of byte-SIMD
  // and 16x2 arithmetic (VABSDIFF4, VIMNMX.U16x2, plain adds on 16-bit lanes
  // that cannot carry); otherwise sample by sample.
  __device__ __forceinline__ void word4(uint32_t cw, uint32_t pw, bool hp, bool track) {
    const uint32_t a4 = __byte_perm(cw, (uint32_t)a, 0x2104);  // left neighbours [a, x0, x1, x2]
    const uint32_t c4 = __byte_perm(pw, (uint32_t)c, 0x2104);  // above-left [c, p0, p1, p2]
    const uint32_t z = (a4 ^ pw) | (pw ^ c4);                   // a zero byte: a == b == c there
    if (!hp || inrun || ((z - 0x01010101u) & ~z & 0x80808080u)) {
#pragma unroll 1
      for (int k = 0; k < 4; k++) {
        sample((int)(cw & 0xFF), (int)(pw & 0xFF), hp, track);
        cw >>= 8;
        pw >>= 8;
      }
      return;
    }
    const uint32_t d1 = __vabsdiffu4(a4, c4), d2 = __vabsdiffu4(c4, pw);
    uint32_t sy[2];
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      const uint32_t sel = hh ? 0x4342u : 0x4140u;  // bytes 2hh, 2hh + 1 -> 16-bit lanes
      const uint32_t x = __byte_perm(cw, 0u, sel), la = __byte_perm(a4, 0u, sel);
      const uint32_t lb = __byte_perm(pw, 0u, sel), lc = __byte_perm(c4, 0u, sel);
      // g = |a - c| + |c - b| (>= 1 here); ctx = 1 + [g > 2] + [g > 8] from min(g, 9)
      const uint32_t gm = vmin_u16x2(__byte_perm(d1, 0u, sel) + __byte_perm(d2, 0u, sel), 0x00090009u);
      const uint32_t f1 = (gm + 0x000D000Du) & 0x00100010u;  // bit 4 of a lane: g > 2
      const uint32_t f2 = (gm + 0x00070007u) & 0x00100010u;  // g > 8
      fge2 += f1;
      fge3 += f2;
      // MED = mn + mx - clamp(c, mn, mx); r = x - MED, low byte of each lane
      const uint32_t mx = vmax_u16x2(la, lb), mn = vmin_u16x2(la, lb);
      const uint32_t cl = vmax_u16x2(mn, vmin_u16x2(lc, mx));
      const uint32_t r = x + cl + 0x04000400u - mn - mx;
      // u = 2r or -2r - 1 (r a signed byte), ctx << 8 beside it
      const uint32_t sgn = (r >> 7) & 0x00010001u;
      const uint32_t hi = sgn * 0xFFu + (f1 + f2) * 16u + 0x01000100u;
      sy[hh] = ((r << 1) & 0x00FE00FEu) ^ hi;
    }
    put4(sy[0], sy[1]);
    if (track && !brk) {
      const uint32_t e = cw ^ a4;  // nonzero byte: x != a (E false)
      if (e) {
        const int k = (__ffs((int)e) - 1) >> 3;
        brk = true;
        cov = nsamp + k;
        brk_i = i - 3 + k;  // symbols up to and including sample k
      }
    }
    nfast += 4;
    nsamp += 4;
    c = (int)(pw >> 24);
    a = (int)(cw >> 24);
  }
  // [x0, x1) of row `cur` (prev: the row above, or nullptr); with `track` the
  // RowTrack facts are recorded
  __device__ __forceinline__ void run(const uint8_t* cur, const uint8_t* prev, int x0, int x1, bool track) {
    const bool hp = prev != nullptr;
    const uint8_t* pv = hp ? prev : cur;
    int x = x0;
    // 16 samples per 128-bit load when the rows are aligned (x0 is a multiple of 16)
    if (((reinterpret_cast<uintptr_t>(cur + x0) | reinterpret_cast<uintptr_t>(pv + x0)) & 15) == 0) {
#pragma unroll 1
      for (; x + 16 <= x1; x += 16) {
        uint4 c4 = __ldg(reinterpret_cast<const uint4*>(cur + x));
        uint4 p4 = __ldg(reinterpret_cast<const uint4*>(pv + x));
#pragma unroll 1
        for (int q = 0; q < 4; q++) {
          word4(c4.x, p4.x, hp, track);
          c4.x = c4.y, c4.y = c4.z, c4.z = c4.w;
          p4.x = p4.y, p4.y = p4.z, p4.z = p4.w;
        }
        fold();
      }
    }
#pragma unroll 1
    for (; x < x1; x++) {
      sample(__ldg(cur + x), __ldg(pv + x), hp, track);
      fold();
    }
  }
};

// The automaton's effect across one segment, as a function of the entry state:
// entering free -> (f_in, f_L) whatever the count; entering inside a run of L
// -> (true, L + cov) when the run covers the whole segment (full), otherwise
// the run ends inside and the exit is (r_in, r_L).  These compose, so a warp
// scan gives every segment its entry state.
struct SegFn {
  bool f_in, full, r_in;
  int f_L, cov, r_L;
};

__device__ __forceinline__ SegFn segfn_identity() { return SegFn{false, true, false, 0, 0, 0}; }

__device__ __forceinline__ void segfn_apply(const SegFn& f, bool& in, int& L) {
  if (!in) {
    in = f.f_in;
    L = f.f_L;
  } else if (f.full) {
    L += f.cov;
  } else {
    in = f.r_in;
    L = f.r_L;
  }
}

__device__ __forceinline__ SegFn segfn_then(const SegFn& f, const SegFn& g) {  // f, then g
  SegFn h;
  h.f_in = f.f_in;
  h.f_L = f.f_L;
  segfn_apply(g, h.f_in, h.f_L);
  if (f.full) {
    h.full = g.full;
    h.cov = f.cov + g.cov;
    h.r_in = g.r_in;
    h.r_L = g.r_L;
  } else {
    h.full = false;
    h.cov = 0;
    h.r_in = f.r_in;
    h.r_L = f.r_L;
    segfn_apply(g, h.r_in, h.r_L);
  }
  return h;
}


__device__ __forceinline__ SegFn shfl_up_segfn(const SegFn& f, int d) {
  const unsigned bits = (unsigned)f.f_in | ((unsigned)f.full << 1) | ((unsigned)f.r_in << 2);
  const unsigned ob = __shfl_up_sync(0xffffffffu, bits, d);
  SegFn g;
  g.f_in = ob & 1;
  g.full = (ob >> 1) & 1;
  g.r_in = (ob >> 2) & 1;
  g.f_L = __shfl_up_sync(0xffffffffu, f.f_L, d);
  g.cov = __shfl_up_sync(0xffffffffu, f.cov, d);
  g.r_L = __shfl_up_sync(0xffffffffu, f.r_L, d);
  return g;
}

// segments per row of a plane of width w: the power of two (dividing 32) that
// brings segments to at most segw samples (ChainTab::plane_segw, chosen per
// launch so that the tiles fill the GPU)
__host__ __device__ __forceinline__ int plane_segs(int w, int segw) { return plane_row_segments(w, segw); }

__host__ __device__ __forceinline__ int plane_seg_width(int w, int segw) {  // multiple of 16
  const int s = plane_segs(w, segw);
  return ((w + s - 1) / s + 15) / 16 * 16;
}

// symbol q of a lane's slab
__device__ __forceinline__ uint32_t slab_symbol(const uint4* slab, int q) {
  const uint4 w = slab[(q >> 3) * 32];
  const int j = q & 7;
  const uint32_t wd = j < 2 ? w.x : (j < 4 ? w.y : (j < 6 ? w.z : w.w));
  return (j & 1) ? (wd >> 16) : (wd & 0xFFFFu);
}

// A lane's symbols: the slab's [start, n), after (for a segment entered inside
// a run) the run's chunks of run_len samples and the symbol `head` (>= 0) of the
// sample that ended it.
struct PlaneBufGen {
  static constexpr bool kStaticCtx = false;
  uint4* slab;  // this lane's chunk 0
  int n;        // symbols in the slab
  int start;    // first slab symbol coded
  int run_len;  // < 0: no chunks
  int head;     // < 0: none
  template <class F>
  __device__ __forceinline__ void for_each(F&& f) const {
    int i = 0;
    if (run_len >= 0) {
      int L = run_len;
      for (;;) {
        const int ch = L >= 255 ? 255 : L;
        f(i++, kRunCtx, ch, 0, 0u);
        L -= ch;
        if (ch < 255) break;
      }
    }
    if (head >= 0) f(i++, (head >> 8) & 7, head & 0xFF, 0, 0u);
    for (int q0 = start & ~7; q0 < n; q0 += 8) {
      SymChunk ch;
      ch.load(slab[(q0 >> 3) * 32]);
      const int m = min(8, n - q0);
#pragma unroll 1  // compact: the kernel's hot code is at the edge of the instruction cache
      for (int j = 0; j < m; j++) {
        const uint32_t sy = ch.pop();
        if (q0 + j >= start) f(i++, (int)((sy >> 8) & 7), (int)(sy & 0xFF), 0, 0u);
      }
    }
  }
};


#ifdef HDLL_PLANE_MINB  // experiment builds: resident CTAs per SM asked of ptxas
#define HDLL_PLANE_LB 128, HDLL_PLANE_MINB
#else
#define HDLL_PLANE_LB 128, 8  // 64 registers, 8 CTAs per SM (-0.12 ms against 72 registers, 7 CTAs)
#endif
#ifdef HDLL_DCT_MINB
#define HDLL_DCT_LB 128, HDLL_DCT_MINB
#else
#define HDLL_DCT_LB 128
#endif

// grid-persistent, 4 warps per CTA, each warp's context state in shared memory
template <bool kCM>
__global__ void __launch_bounds__(HDLL_PLANE_LB) k_entropy_plane(const ImgDesc* __restrict__ descs, ChainTab ct, uint4* symbuf,
                                                       int cap_chunks, uint32_t* wordbuf) {
  __shared__ __align__(16) uint8_t smem_pl[4 * lane_state_bytes(5)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const LaneState ls = carve_state(smem_pl + warp * lane_state_bytes(5), 5);
  uint4* slab = symbuf + ((long long)blockIdx.x * 4 + warp) * cap_chunks * 32 + lane;
  uint32_t* scr = wordbuf + ((long long)blockIdx.x * 4 + warp) * cap_chunks * 8 * 32 + lane;  // <= 1 word per symbol
  int chain;
  long long tin, g;
  while (next_tile<kCM>(ct, &chain, &tin, &g)) {
    const ImgDesc& d = descs[ct.img[chain]];
    const int kind = ct.kind[chain];
    const int S = plane_segs(d.w, ct.plane_segw), wseg = plane_seg_width(d.w, ct.plane_segw);
    const long long r = tin * (kPlaneTileRows / S) + lane / S;  // row of the chain
    const int sg = lane & (S - 1);
    const int x0 = min(d.w, sg * wseg), x1 = min(d.w, x0 + wseg);
    const bool live = r < ct.units[chain];
    const uint8_t* src = kind == 1 ? d.e_plane : d.res_planes + (long long)(kind - 2) * d.n;
    const long long y = ct.first[chain] + (live ? r : 0);  // row in the image arrays
    const uint8_t* cur = src + y * d.w;
    const uint8_t* prev = y > 0 ? cur - d.w : nullptr;
    // Every segment is coded entered free; a segment that continues a run
    // from the previous ones (segmented scan of the segments' automaton
    // functions, derived from the same pass) then swaps the free coding's
    // symbols up to its first run-ending sample for the run's chunks.
    RowTrack trk;
    trk.brk = false;
    trk.cov = 0;
    trk.brk_i = 0;
    trk.out_in = false;
    trk.out_L = 0;
    int cnt[5] = {0, 0, 0, 0, 0};
    int n = 0;
    if (live) {
      SegGen sg_;
      sg_.a = x0 > 0 ? cur[x0 - 1] : (prev ? __ldg(prev) : 128);
      sg_.c = x0 > 0 ? (prev ? prev[x0 - 1] : sg_.a) : sg_.a;  // above-left (the above sample at x = 0)
      sg_.inrun = false;
      sg_.L = 0;
      sg_.i = 0;
      sg_.sp = slab;
      sg_.cpk = 0;
      sg_.fge2 = sg_.fge3 = 0;
      sg_.nfast = 0;
#pragma unroll
      for (int c = 0; c < 5; c++) sg_.cnt[c] = 0;
      sg_.brk = false;
      sg_.cov = sg_.brk_i = sg_.nsamp = 0;
      const bool track = S > 1;
      sg_.run(cur, prev, x0, x1, track);
      trk.brk = sg_.brk;
      trk.cov = sg_.brk ? sg_.cov : x1 - x0;
      trk.brk_i = sg_.brk_i;
      trk.out_in = sg_.inrun;
      trk.out_L = sg_.L;
      if (sg_.inrun && x1 == d.w) sg_.run_chunks();  // a run reaching the row end
      n = sg_.i;
      if (n & 7) {
        sg_.ch.align(n & 7);
        *sg_.sp = sg_.ch.word();
      }
#pragma unroll
      for (int c = 0; c < 5; c++) cnt[c] = sg_.cnt[c];
    }
    PlaneBufGen gen{slab, n, 0, -1, -1};
    if (S > 1) {
      SegFn f = segfn_identity();
      if (live) {
        f.f_in = trk.out_in;
        f.f_L = trk.out_L;
        f.full = !trk.brk;
        f.cov = trk.cov;
        f.r_in = trk.out_in;
        f.r_L = trk.out_L;
      }
      for (int dd = 1; dd < S; dd <<= 1) {
        const SegFn o = shfl_up_segfn(f, dd);
        if (sg >= dd) f = segfn_then(o, f);
      }
      const SegFn ex = shfl_up_segfn(f, 1);
      bool in0 = false;
      int L0 = 0;
      if (sg > 0) segfn_apply(ex, in0, L0);
      if (live && in0) {  // entered inside a run of L0 samples
        const int run = L0 + trk.cov;
        const int upto = trk.brk ? trk.brk_i : n;  // free symbols replaced
        for (int q = 0; q < upto; q++) cnt[(slab_symbol(slab, q) >> 8) & 7]--;
        const bool chunks = trk.brk || x1 == d.w;  // the run ends here (or with the row)
        if (chunks) cnt[kRunCtx] += run / 255 + 1;
        gen.start = upto;
        gen.run_len = chunks ? run : -1;
        if (trk.brk) {
          gen.head = (int)slab_symbol(slab, trk.brk_i - 1);
          cnt[(gen.head >> 8) & 7]++;
        }
      }
    }
#ifdef HDLL_EXP_COUNT_ONLY  // timing experiment: the generation pass alone
    if (cnt[0] == -1) atomicOr(d.status, 1u);
#else
    run_tile<5, 5, kCM>(ct, chain, tin, g, 0, gen, cnt, ls, d.status, scr, cap_chunks * 8);
#endif
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// DCT coder: tile = 32 lanes x dct_bpl consecutive blocks of one component
// ---------------------------------------------------------------------------
// a block's code: <= 544 bytes (dct_chain_cap) = 136 words
constexpr int kDctScrWords = 136;

template <bool kCM>
__global__ void __launch_bounds__(HDLL_DCT_LB) k_entropy_dct(const ImgDesc* __restrict__ descs, ChainTab ct, uint32_t* wordbuf) {
  __shared__ __align__(16) uint8_t smem_dct[4 * lane_state_bytes(3)];
  __shared__ unsigned long long s_nzm[4][kDctMaxBlocksPerLane * 32];
  __shared__ unsigned s_dcu[4][kDctMaxBlocksPerLane * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const LaneState ls = carve_state(smem_dct + warp * lane_state_bytes(3), 3);
  const int bpl = ct.dct_bpl;
  uint32_t* scr = wordbuf + ((long long)blockIdx.x * 4 + warp) * kDctScrWords * bpl * 32 + lane;
  int chain;
  long long tin, g;
  while (next_tile<kCM>(ct, &chain, &tin, &g)) {
    const ImgDesc& d = descs[ct.img[chain]];
    const long long units = ct.units[chain];
    const long long per = 32LL * bpl;
    const long long tpc = (units + per - 1) / per;
    const int comp = ct.comp[chain];  // >= 0: that component; -1: Y, Cb, Cr; -2: Cb, Cr
    const int ci = comp >= 0 ? comp : (comp == -2 ? 1 : 0) + (int)(tin / tpc);
    const long long tl = comp >= 0 ? tin : tin % tpc;
    const long long u0 = tl * per + (long long)lane * bpl;  // the lane's first block in the chain
    const int nb = (int)max(0LL, min((long long)bpl, units - u0));
    const long long bi0 = ct.first[chain] + u0;             // ... in the image arrays
    int cnt[3] = {0, 0, 0};
    for (int k = 0; k < nb; k++) {
      const long long bi = bi0 + k;
      const int16_t* z = d.zz + ((long long)ci * d.nblocks + bi) * 64;
      // nonzero mask of the 64 zigzag coefficients, 128-bit loads
      const uint4* z4 = reinterpret_cast<const uint4*>(z);
      unsigned long long nzm = 0;
      int dc = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        uint4 v = z4[q];
        uint32_t ws[4] = {v.x, v.y, v.z, v.w};
        if (q == 0) dc = (int)(int16_t)(ws[0] & 0xFFFF);
#pragma unroll
        for (int r = 0; r < 4; r++) {
          nzm |= (unsigned long long)((ws[r] & 0xFFFFu) != 0) << (q * 8 + r * 2);
          nzm |= (unsigned long long)((ws[r] >> 16) != 0) << (q * 8 + r * 2 + 1);
        }
      }
      nzm &= ~1ULL;
      const int prev_dc = bi > 0 ? d.zz[((long long)ci * d.nblocks + bi - 1) * 64] : 0;
      const int dv = dc - prev_dc;
      s_nzm[warp][k * 32 + lane] = nzm;
      s_dcu[warp][k * 32 + lane] = dv >= 0 ? 2u * dv : (unsigned)(-2 * dv - 1);
      const int nnz = __popcll(nzm);
      cnt[0] += 1;
      cnt[1] += nnz + ((nzm >> 63) ? 0 : 1);  // runs + EOB (absent when position 63 is coded)
      cnt[2] += nnz;
    }
    const DctRunGen gen{nb > 0 ? d.zz + ((long long)ci * d.nblocks + bi0) * 64 : nullptr, &s_nzm[warp][lane],
                        &s_dcu[warp][lane], nb};
    run_tile<3, 6, kCM>(ct, chain, tin, g, ci == 0 ? 0 : 3, gen, cnt, ls, d.status, scr, kDctScrWords * bpl);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Fix-up: merge the words shared between tiles.  Word w belongs to the tile
// holding its first bit; that tile's tail plus the heads of the following
// tiles that start inside w (several, if tiles are tiny) are OR-ed once.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_chain(const ChainTab& ct, long long g) {
  int lo = 0, hi = ct.nchains;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (ct.tile_base[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_entropy_fixup(ChainTab ct) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ct.ntiles) return;
  const int chain = find_chain(ct, g);
  if (ct.chain_mode && chain_mode<true>(ct, chain) != 0) return;
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

// ---------------------------------------------------------------------------
// mode 2: compose every chain's tile aggregates (oldest first) into out_map.
// One warp per (chain, context): lanes compose contiguous runs, then the warp.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) k_chain_maps(ChainTab ct) {
  const int chain = blockIdx.x, c = blockIdx.y, lane = threadIdx.x;
  if ((ct.chain_mode ? chain_mode<true>(ct, chain) : ct.mode) != 2) return;
  const long long t0 = ct.tile_base[chain], nt = ct.tile_base[chain + 1] - t0;
  const long long per = (nt + 31) / 32;
  AMap m = amap_identity();
  for (long long j = lane * per; j < min(nt, (lane + 1) * per); j++) m = amap_then(m, ct.maps[(t0 + j) * kMaxCtx + c]);
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {  // lane 0 holds the oldest run: compose x then (lane + d)
    AMap y;
    y.c = __shfl_down_sync(0xffffffffu, m.c, d);
    y.s = __shfl_down_sync(0xffffffffu, m.s, d);
    y.t = __shfl_down_sync(0xffffffffu, m.t, d);
    if (lane + d < 32) m = amap_then(m, y);
  }
  if (lane == 0) ct.out_map[chain * kMaxCtx + c] = m;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static long long dct_grid(const ChainTab& ct) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_entropy_dct<false>, 128, 0);
  long long blocks = (long long)num_sms() * (per_sm > 0 ? per_sm : 1);
  const long long need = (ct.ntiles + 3) / 4;
  return blocks < need ? blocks : need;
}

size_t dct_scratch_bytes(const ChainTab& ct) {
  if (ct.ntiles <= 0) return 0;
  return (size_t)dct_grid(ct) * 4 * 32 * kDctScrWords * ct.dct_bpl * sizeof(uint32_t);
}

void launch_entropy_dct(const ImgDesc* d_descs, const ChainTab& ct, void* scratch, cudaStream_t st) {
  if (ct.ntiles <= 0) return;
  if (ct.chain_mode) k_entropy_dct<true><<<(unsigned)dct_grid(ct), 128, 0, st>>>(d_descs, ct, (uint32_t*)scratch);
  else k_entropy_dct<false><<<(unsigned)dct_grid(ct), 128, 0, st>>>(d_descs, ct, (uint32_t*)scratch);
}

static long long plane_grid(const ChainTab& ct) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_entropy_plane<false>, 128, 0);
  long long blocks = (long long)num_sms() * (per_sm > 0 ? per_sm : 1);
  const long long need = (ct.ntiles + 3) / 4;
  return blocks < need ? blocks : need;
}

// a segment: <= 2 symbols per sample, plus the 255-chunks of a run that may
// have begun anywhere earlier in the row
static int plane_cap_chunks(int max_w, int segw) {
  int ws = segw + 16;
  if (ws > max_w) ws = max_w;
  return (2 * ws + max_w / 255 + 16) / 8 + 1;
}

// per warp: the symbol slab (16 B per 8 symbols) and the code words (<= 4 B per symbol)
static size_t plane_warp_bytes(int cap_chunks) { return (size_t)32 * cap_chunks * (sizeof(uint4) + 8 * sizeof(uint32_t)); }

size_t plane_scratch_bytes(const ChainTab& ct, int max_w) {
  if (ct.ntiles <= 0) return 0;
  return (size_t)plane_grid(ct) * 4 * plane_warp_bytes(plane_cap_chunks(max_w, ct.plane_segw));
}

void launch_entropy_plane(const ImgDesc* d_descs, const ChainTab& ct, int max_w, void* scratch, cudaStream_t st) {
  if (ct.ntiles <= 0) return;
  const long long grid = plane_grid(ct);
  const int cc = plane_cap_chunks(max_w, ct.plane_segw);
  uint4* slabs = (uint4*)scratch;
  uint32_t* words = (uint32_t*)(slabs + grid * 4 * 32 * cc);
  if (ct.chain_mode) k_entropy_plane<true><<<(unsigned)grid, 128, 0, st>>>(d_descs, ct, slabs, cc, words);
  else k_entropy_plane<false><<<(unsigned)grid, 128, 0, st>>>(d_descs, ct, slabs, cc, words);
}

void launch_entropy_fixup(const ChainTab& ct, cudaStream_t st) {
  if (ct.ntiles <= 0) return;
  if (ct.modes_present & 4) k_chain_maps<<<dim3(ct.nchains, kMaxCtx), 32, 0, st>>>(ct);
  if (ct.modes_present & 1) k_entropy_fixup<<<(unsigned)((ct.ntiles + 255) / 256), 256, 0, st>>>(ct);
}

}  // namespace hdll
