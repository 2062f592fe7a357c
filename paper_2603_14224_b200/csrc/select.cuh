// Block-/group-wide selection helpers shared by the decode kernels and the generic top-k.
// Helpers are templated on a thread group: the whole 256-thread CTA (Cta256) or a
// 256-thread slice of a larger CTA synchronised by a named barrier (NamedGroup).
#pragma once
#include "common.cuh"

namespace sikv {

constexpr int DT = 256;            // threads per selection / decode group
constexpr int DW = DT / 32;

struct Cta256 {
  static __device__ __forceinline__ int tid() { return threadIdx.x; }
  static __device__ __forceinline__ void sync() { __syncthreads(); }
};
template <int ID, int BASE>
struct NamedGroup {                // threads [BASE, BASE + 256) of the CTA, barrier ID
  static __device__ __forceinline__ int tid() { return (int)threadIdx.x - BASE; }
  static __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, 256;\n" ::"n"(ID) : "memory"); }
};

// Cross-CTA exchange policy for split units (a CTA cluster sharing one unit).  NoX: the
// group owns the whole unit, every "global" value is the local one.  Each hook is called by
// every thread of the group after the group has synchronised on the local value.
struct NoX {
  static constexpr bool kCluster = false;
  __device__ __forceinline__ void sample(int&, uint32_t&, uint32_t&) const {}
  __device__ __forceinline__ void hist256(const int*&, const uint32_t*&) const {}
  __device__ __forceinline__ void counts(int&, int&, bool&) const {}
  template <int NBINT = 2048>
  __device__ __forceinline__ const int* hist4k(const int* h) const { return h; }
  __device__ __forceinline__ uint32_t maxu(uint32_t v) const { return v; }
};

// ---------------------------------------------------------------- small group utilities
struct Misc {                      // scalars in shared memory
  int ncand, nsv, digit, rem_sel, cnt_above, total, fb, bad;
  uint32_t tau, maxx;
  int wsum[DW * 2];
  int wcnt[DW];                    // per-warp candidate counts
};

template <class Grp = Cta256>
__device__ __forceinline__ void block_exscan2(int a, int b, int& ea, int& eb, int& ta, int& tb, int* wsum) {
  const int t = Grp::tid(), lane = t & 31, warp = t >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += xa; ib += xb; }
  }
  if (lane == 31) { wsum[warp] = ia; wsum[DW + warp] = ib; }
  Grp::sync();
  int pa = 0, pb = 0, sa = 0, sb = 0;
  for (int w = 0; w < DW; ++w) {
    if (w < warp) { pa += wsum[w]; pb += wsum[DW + w]; }
    sa += wsum[w]; sb += wsum[DW + w];
  }
  ea = pa + ia - a; eb = pb + ib - b; ta = sa; tb = sb;
  Grp::sync();
}

// warp-aggregated shared-memory histogram increment (bin < 0 = no-op)
__device__ __forceinline__ void hist_add(int* hist, int bin) {
  unsigned peers = __match_any_sync(0xffffffffu, bin);
  int leader = __ffs(peers) - 1;
  if (bin >= 0 && (int)(threadIdx.x & 31) == leader) atomicAdd(&hist[bin], __popc(peers));
}

// warp 0 picks the digit whose cumulative count (from the top bin) reaches `rem` (256 bins)
__device__ __forceinline__ void pick_digit(const int* hist, Misc* ms) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int loc[8], s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { loc[i] = hist[255 - 8 * lane - i]; s += loc[i]; }
  int inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  const int exc = inc - s, rem = ms->rem_sel;
  if (exc < rem && rem <= inc) {
    int c = exc;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (c < rem && rem <= c + loc[i]) { ms->digit = 255 - 8 * lane - i; ms->cnt_above = c; }
      c += loc[i];
    }
  }
}

// ---------------------------------------------------------------- 11-bit radix k-th selection
constexpr int RB = 11;              // digit bits per pass
constexpr int NBIN = 1 << RB;       // 2048 bins; thread t owns bins [NBIN-8(t+1), NBIN-8t)

// Group-wide: choose the digit whose descending cumulative count reaches ms->rem_sel.
template <class Grp = Cta256, int NBINT = NBIN>
__device__ __forceinline__ void pick_digit_big(const int* hist, Misc* ms) {
  static_assert(NBINT >= DT && NBINT % DT == 0, "bins per thread");
  const int tid = Grp::tid();
  constexpr int PER = NBINT / DT;
  const int top = NBINT - 1 - PER * tid;          // this thread owns bins top, top-1, ..., top-PER+1
  int s = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) s += hist[top - ((i + tid) & (PER - 1))];   // rotated: no bank conflicts
  int exc, d0, tot, d1;
  block_exscan2<Grp>(s, 0, exc, d0, tot, d1, ms->wsum);
  const int rem = ms->rem_sel;
  if (exc < rem && rem <= exc + s) {
    int c = exc;
    for (int i = 0; i < PER; ++i) {
      const int h = hist[top - i];
      if (c < rem && rem <= c + h) { ms->digit = top - i; ms->cnt_above = c; break; }
      c += h;
    }
  }
  Grp::sync();
}

// Exact k-th largest of a multiset of 32-bit values x (all <= maxx).  `each(f)` must call
// f(x) once per item on the calling thread (every thread of the group calls each()).
// Returns the k-th value and how many items equal to it belong to the top `rank` (ties
// are then resolved by index by the caller).  hist must hold NBINT + 33 ints (NBINT = 2^digit
// bits: 2048 by default, 512 for the two-kernel path's selection groups).
template <class Grp = Cta256, class Xch = NoX, int NBINT = NBIN, typename Each>
__device__ __forceinline__ void radix_kth(Each each, uint32_t maxx, int rank, int* hist, Misc* ms,
                                          uint32_t& kth, int& need_eq, const Xch& xch = Xch()) {
  const int tid = Grp::tid();
  const int nbits = maxx ? 32 - __clz(maxx) : 0;
  constexpr int RBT = __builtin_ctz(NBINT);
  int* list = hist + NBINT;          // up to 32 items of a small boundary bin (+ counter)
  if (tid == 0) ms->rem_sel = rank;
  uint32_t prefix = 0;
  int shift = nbits;
  Grp::sync();
  while (shift > 0) {
    const int dbits = shift >= RBT ? RBT : shift;
    const int hi = shift;            // bits >= hi are already fixed in prefix
    shift -= dbits;
    for (int i = tid; i < NBINT; i += DT) hist[i] = 0;
    if (tid == 0) list[32] = 0;
    Grp::sync();
    const uint32_t want = hi >= 32 ? 0u : (prefix >> hi);
    const int sh = shift;
    each([&](uint32_t x) {
      if ((hi >= 32 ? 0u : (x >> hi)) == want) atomicAdd(&hist[(x >> sh) & (NBINT - 1)], 1);
    });
    Grp::sync();
    const int* mh = xch.template hist4k<NBINT>(hist);   // cluster: the sum of every CTA's histogram
    pick_digit_big<Grp, NBINT>(mh, ms);
    const uint32_t d = (uint32_t)ms->digit;
    prefix |= d << shift;
    const int nb = mh[d];
    Grp::sync();
    if (tid == 0) ms->rem_sel -= ms->cnt_above;
    Grp::sync();
    if (!Xch::kCluster && shift > 0 && nb <= 32) {
      // finish inside one warp: exact rank among the few items of the boundary bin
      const uint32_t w2 = prefix >> shift;
      each([&](uint32_t x) {
        if ((x >> shift) == w2) list[atomicAdd(&list[32], 1)] = (int)x;
      });
      Grp::sync();
      if (tid < 32) {
        const uint32_t v = tid < nb ? (uint32_t)list[tid] : 0u;
        int gt = 0, eqc = 0;
        for (int j = 0; j < nb; ++j) {
          const uint32_t o = (uint32_t)list[j];
          gt += o > v;
          eqc += o == v;
        }
        const int rem = ms->rem_sel;
        __syncwarp();
        if (tid < nb && gt < rem && rem <= gt + eqc) { ms->tau = v; ms->digit = rem - gt; }
      }
      Grp::sync();
      kth = ms->tau;
      need_eq = ms->digit;
      Grp::sync();
      return;
    }
  }
  kth = prefix;
  need_eq = ms->rem_sel;
  Grp::sync();
}

}  // namespace sikv
