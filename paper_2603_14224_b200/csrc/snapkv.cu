// SnapKV-style window sinks on the GPU (cache.py:185-209, the query_window branch of prefill,
// cache.py:249-252), batched over units, in float64 like the reference:
//
//   logits[t][j] = (K'[t] . W[j]) / sqrt(D)            K' = K - mu (float64, frozen prefill mu)
//   weights      = column softmax of logits over t     (max-subtracted)
//   votes[t]     = sum_j weights[t][j]                 (numpy's 8-accumulator pairwise order)
//   pooled       = maximum_filter1d(votes, 7, mode="nearest")
//   sinks        = sorted(stable top-count of pooled)  (ties -> lower index; generic.cu topk)
//
//   snap_logits_kernel  one 256-thread CTA per 512 tokens of a unit: the window queries in
//                       shared memory (float64, broadcast reads), each thread two tokens x 16
//                       columns per pass, logits stored (float64) plus the CTA's per-column
//                       (max, sum of exp) partials;
//   snap_votes_kernel   merges the partials per column, then votes and the max-pool.
// Arithmetic: the dot products and sums run in float64 in a fixed order that differs from
// the reference's BLAS / pairwise order by rounding only (~1e-16 relative); sink sets are
// exact unless two distinct pooled votes at the count boundary are that close (max-pool
// plateaus are exact copies and tie-break identically).
#include "common.cuh"
#include <math.h>
#include <algorithm>

namespace sikv {

constexpr int SNAP_T = 256;          // threads per CTA
constexpr int SNAP_TOK = 512;        // tokens per CTA (2 per thread)
constexpr int SNAP_COLS = 16;        // window columns per pass

__global__ void __launch_bounds__(SNAP_T) snap_logits_kernel(const void* __restrict__ keys, int dt, int64_t L, int D,
                                                             const double* __restrict__ mu64,
                                                             const double* __restrict__ win, int w,
                                                             double* __restrict__ logits, double* __restrict__ part) {
  extern __shared__ __align__(16) double snap_sm[];
  double* Ws = snap_sm;                    // [w][D]
  double* mus = Ws + (size_t)w * D;        // [D]
  double* red = mus + D;                   // [8 warps][2][SNAP_COLS]
  const int64_t u = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < w * D; i += SNAP_T) Ws[i] = win[(int64_t)u * w * D + i];
  for (int i = tid; i < D; i += SNAP_T) mus[i] = mu64[u * D + i];
  __syncthreads();
  const double rs = 1.0 / sqrt((double)D);
  const int64_t tbase = (int64_t)blockIdx.x * SNAP_TOK;
  const int64_t t0 = tbase + tid, t1 = tbase + tid + SNAP_T;
  const bool v0 = t0 < L, v1 = t1 < L;
  const int nchunks = gridDim.x;
  for (int j0 = 0; j0 < w; j0 += SNAP_COLS) {
    const int nc = min(SNAP_COLS, w - j0);
    double a0[SNAP_COLS], a1[SNAP_COLS];
#pragma unroll
    for (int j = 0; j < SNAP_COLS; ++j) { a0[j] = 0.0; a1[j] = 0.0; }
    for (int d = 0; d < D; d += 4) {
      double k0[4], k1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        k0[i] = v0 ? load_in(keys, dt, (u * L + t0) * D + d + i) - mus[d + i] : 0.0;
        k1[i] = v1 ? load_in(keys, dt, (u * L + t1) * D + d + i) - mus[d + i] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < SNAP_COLS; ++j) {
        if (j < nc) {
          const double* wr = Ws + (size_t)(j0 + j) * D + d;
          const double2 wa = *reinterpret_cast<const double2*>(wr);
          const double2 wb = *reinterpret_cast<const double2*>(wr + 2);
          a0[j] = fma(k0[3], wb.y, fma(k0[2], wb.x, fma(k0[1], wa.y, fma(k0[0], wa.x, a0[j]))));
          a1[j] = fma(k1[3], wb.y, fma(k1[2], wb.x, fma(k1[1], wa.y, fma(k1[0], wa.x, a1[j]))));
        }
      }
    }
    // logits, then this CTA's per-column max and sum of exp(logit - max)
#pragma unroll
    for (int j = 0; j < SNAP_COLS; ++j) {
      if (j >= nc) break;
      const double l0 = a0[j] * rs, l1 = a1[j] * rs;
      if (v0) logits[(u * L + t0) * w + j0 + j] = l0;
      if (v1) logits[(u * L + t1) * w + j0 + j] = l1;
      double m = fmax(v0 ? l0 : -INFINITY, v1 ? l1 : -INFINITY);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp * 2 * SNAP_COLS + j] = m;
      a0[j] = l0;
      a1[j] = l1;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SNAP_COLS; ++j) {
      if (j >= nc) break;
      double M = -INFINITY;
      for (int wi = 0; wi < SNAP_T / 32; ++wi) M = fmax(M, red[wi * 2 * SNAP_COLS + j]);
      double s = (v0 ? exp(a0[j] - M) : 0.0) + (v1 ? exp(a1[j] - M) : 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp * 2 * SNAP_COLS + SNAP_COLS + j] = s;
    }
    __syncthreads();
    if (tid < nc) {
      double M = -INFINITY, s = 0.0;
      for (int wi = 0; wi < SNAP_T / 32; ++wi) M = fmax(M, red[wi * 2 * SNAP_COLS + tid]);
      for (int wi = 0; wi < SNAP_T / 32; ++wi) s += red[wi * 2 * SNAP_COLS + SNAP_COLS + tid];
      double* p = part + ((u * nchunks + blockIdx.x) * w + j0 + tid) * 2;
      p[0] = M;
      p[1] = s;
    }
    __syncthreads();
  }
}

// per-column totals from the CTA partials, then votes (8-accumulator pairwise sum over the
// window columns, numpy's order for a contiguous row) for SNAP_T tokens per CTA
__global__ void __launch_bounds__(SNAP_T) snap_votes_kernel(const double* __restrict__ logits,
                                                            const double* __restrict__ part, int64_t L, int w,
                                                            int nchunks, double* __restrict__ votes) {
  __shared__ double colM[64], colS[64];
  const int64_t u = blockIdx.y;
  const int tid = threadIdx.x;
  if (tid < w) {
    double M = -INFINITY;
    for (int c = 0; c < nchunks; ++c) M = fmax(M, part[((u * nchunks + c) * w + tid) * 2]);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      const double* p = part + ((u * nchunks + c) * w + tid) * 2;
      if (p[1] > 0.0) s += p[1] * exp(p[0] - M);
    }
    colM[tid] = M;
    colS[tid] = s;
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * SNAP_T + tid;
  if (t >= L) return;
  const double* lr = logits + (u * L + t) * w;
  auto wt = [&](int j) { return exp(lr[j] - colM[j]) / colS[j]; };
  double v;
  if (w < 8) {
    v = 0.0;
    for (int j = 0; j < w; ++j) v += wt(j);
  } else {
    double r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = wt(i);
    int j = 8;
    for (; j + 8 <= w; j += 8)
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] += wt(j + i);
    v = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; j < w; ++j) v += wt(j);
  }
  votes[u * L + t] = v;
}

// maximum_filter1d(votes, size=pool, mode="nearest") (edge values replicated)
__global__ void snap_pool_kernel(const double* __restrict__ votes, int64_t L, int pool, double* __restrict__ pooled) {
  const int64_t u = blockIdx.y;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L) return;
  const int lo = pool / 2, hi = pool - 1 - pool / 2;   // scipy's origin-0 window: [t - lo, t + hi]
  double m = -INFINITY;
  for (int64_t s = t - lo; s <= t + hi; ++s) {
    const int64_t c = s < 0 ? 0 : (s >= L ? L - 1 : s);
    m = fmax(m, votes[u * L + c]);
  }
  pooled[u * L + t] = m;
}

size_t snap_workspace_bytes(int64_t U, int64_t L, int w) {
  const int64_t nch = (L + SNAP_TOK - 1) / SNAP_TOK;
  auto a = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return a((size_t)U * L * w * 8) + a((size_t)U * nch * w * 16) + 2 * a((size_t)U * L * 8);
}

cudaError_t launch_snap_pooled(const void* keys, int dt, int64_t U, int64_t L, int D, const double* mu64,
                               const double* win, int w, int pool, void* workspace, double** pooled_out,
                               cudaStream_t st) {
  auto a = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const int nch = (int)((L + SNAP_TOK - 1) / SNAP_TOK);
  char* p = reinterpret_cast<char*>(workspace);
  double* logits = reinterpret_cast<double*>(p);
  p += a((size_t)U * L * w * 8);
  double* part = reinterpret_cast<double*>(p);
  p += a((size_t)U * nch * w * 16);
  double* votes = reinterpret_cast<double*>(p);
  p += a((size_t)U * L * 8);
  double* pooled = reinterpret_cast<double*>(p);
  const size_t smem = ((size_t)w * D + D + 8 * 2 * SNAP_COLS) * 8;
  cudaError_t e = cudaFuncSetAttribute(snap_logits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  snap_logits_kernel<<<dim3(nch, (unsigned)U), SNAP_T, smem, st>>>(keys, dt, L, D, mu64, win, w, logits, part);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  snap_votes_kernel<<<dim3((unsigned)((L + SNAP_T - 1) / SNAP_T), (unsigned)U), SNAP_T, 0, st>>>(logits, part, L, w,
                                                                                                nch, votes);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  snap_pool_kernel<<<dim3((unsigned)((L + 255) / 256), (unsigned)U), 256, 0, st>>>(votes, L, pool, pooled);
  *pooled_out = pooled;
  return cudaGetLastError();
}

}  // namespace sikv
