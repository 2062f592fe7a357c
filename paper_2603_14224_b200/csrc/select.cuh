// Block-wide selection helpers shared by the fused decode kernel and the generic top-k.
#pragma once
#include "common.cuh"

namespace sikv {

constexpr int DT = 256;            // threads per selection / decode CTA
constexpr int DW = DT / 32;

// ---------------------------------------------------------------- small block utilities
struct Misc {                      // scalars in shared memory
  int ncand, nsv, digit, rem_sel, cnt_above, total, fb;
  uint32_t tau;
  int wsum[DW * 2];
};

__device__ __forceinline__ void block_exscan2(int a, int b, int& ea, int& eb, int& ta, int& tb,
                                              int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += xa; ib += xb; }
  }
  if (lane == 31) { wsum[warp] = ia; wsum[DW + warp] = ib; }
  __syncthreads();
  int pa = 0, pb = 0, sa = 0, sb = 0;
  for (int w = 0; w < DW; ++w) {
    if (w < warp) { pa += wsum[w]; pb += wsum[DW + w]; }
    sa += wsum[w]; sb += wsum[DW + w];
  }
  ea = pa + ia - a; eb = pb + ib - b; ta = sa; tb = sb;
  __syncthreads();
}

// warp-aggregated shared-memory histogram increment (bin < 0 = no-op)
__device__ __forceinline__ void hist_add(int* hist, int bin) {
  unsigned peers = __match_any_sync(0xffffffffu, bin);
  int leader = __ffs(peers) - 1;
  if (bin >= 0 && (int)(threadIdx.x & 31) == leader) atomicAdd(&hist[bin], __popc(peers));
}

// warp 0 picks the digit whose cumulative count (from the top bin) reaches `rem`
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

}  // namespace sikv
