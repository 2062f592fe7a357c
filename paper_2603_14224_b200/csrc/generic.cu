// Reference-layout, float64 kernels behind the per-head drop-in API.
//
// These reproduce the reference's float64 arithmetic in the reference's own order where
// the order decides bits (LUT pairing, numpy pairwise row sums, stable top-k) so that
// build_lut / score_tokens / top_k_select / select_tokens return the reference's exact
// numbers.  The batched hot path is decode.cu; these kernels serve the per-head API and
// the variant modes (any D <= 128, bits 1/2/4/8/16, direct-key mode, sign-only LUT).
#include "common.cuh"
#include "select.cuh"
#include "api_types.cuh"
#include <math.h>
#include <algorithm>

namespace sikv {

// ---------------------------------------------------------------- LUT (retrieval.py:46-62)
__global__ void lut_f64_kernel(const double* __restrict__ q, const double* __restrict__ cent, int G,
                               int sign_only, double* __restrict__ out) {
  const int64_t u = blockIdx.x;
  for (int e = threadIdx.x; e < G * 16; e += blockDim.x) {
    const int g = e >> 4, c = e & 15;
    const double* qq = q + u * G * 4 + 4 * g;
    double r;
    if (sign_only) {
      double p[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) p[i] = ((c >> (3 - i)) & 1) ? qq[i] : -qq[i];
      r = (G == 1) ? __dadd_rn(__dadd_rn(p[0], p[2]), __dadd_rn(p[1], p[3]))
                   : __dadd_rn(__dadd_rn(__dadd_rn(p[0], p[1]), p[2]), p[3]);
    } else {
      const double* cc = cent + (u * G + g) * 64 + 4 * c;
      r = __dadd_rn(__dadd_rn(__dmul_rn(qq[0], cc[0]), __dmul_rn(qq[2], cc[2])),
                    __dadd_rn(__dmul_rn(qq[1], cc[1]), __dmul_rn(qq[3], cc[3])));
    }
    out[u * G * 16 + e] = r;
  }
}

// ---------------------------------------------------------------- scores (retrieval.py:65-77)
// numpy pairwise order for one row of n <= 128 terms.
__device__ __forceinline__ double pairwise_row(const double* x, int n) {
  if (n < 8) {
    double r = x[0];
    for (int i = 1; i < n; ++i) r = __dadd_rn(r, x[i]);
    return r;
  }
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = x[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(a[j], x[i + j]);
  double r = __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                       __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
  for (; i < n; ++i) r = __dadd_rn(r, x[i]);
  return r;
}

__global__ void score_f64_kernel(const double* __restrict__ lut, const uint8_t* __restrict__ codes, int G,
                                 int64_t L, double* __restrict__ out) {
  extern __shared__ double tbl[];
  const int64_t u = blockIdx.y;
  for (int e = threadIdx.x; e < G * 16; e += blockDim.x) tbl[e] = lut[u * G * 16 + e];
  __syncthreads();
  const int rowb = (G + 1) / 2;
  double x[128];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < L; t += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = codes + (u * L + t) * rowb;
    for (int g = 0; g < G; ++g) {
      const int c = (r[g >> 1] >> (4 * (g & 1))) & 15;
      x[g] = tbl[g * 16 + c];
    }
    out[u * L + t] = pairwise_row(x, G);
  }
}

// ---------------------------------------------------------------- exact top-k (retrieval.py:127-161)
// scores (f64 or f32) -> sorted indices of forced U dynamic; forced = the given index list.
// Keys are 64-bit order-preserving transforms; ties resolve to the lower index.
__device__ __forceinline__ uint64_t score_key(const void* s, int is_f32, int64_t i) {
  if (is_f32) {
    uint32_t k = f32_key(reinterpret_cast<const float*>(s)[i]);
    return (uint64_t)k << 32;
  }
  return f64_key(reinterpret_cast<const double*>(s)[i]);
}

__global__ void __launch_bounds__(DT) topk_kernel(const void* __restrict__ scores, int is_f32, int64_t L,
                                                  const int32_t* __restrict__ forced_idx, int F, int k,
                                                  uint32_t* __restrict__ ws, int32_t* __restrict__ out,
                                                  int out_stride, int32_t* __restrict__ counts) {
  __shared__ Misc ms_;
  Misc* ms = &ms_;
  const int tid = threadIdx.x;
  const int64_t u = blockIdx.x;
  const int W = (int)((L + 31) >> 5);
  uint32_t* forced = ws + u * 3 * (int64_t)W;
  uint32_t* gt = forced + W;
  uint32_t* eq = gt + W;
  const void* s = is_f32 ? (const void*)((const float*)scores + u * L) : (const void*)((const double*)scores + u * L);
  for (int i = tid; i < 3 * W; i += DT) forced[i] = 0u;
  __syncthreads();
  for (int j = tid; j < F; j += DT) {
    const int t = forced_idx[u * F + j];
    atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  int nf = 0;
  for (int i = tid; i < W; i += DT) nf += __popc(forced[i]);
  int nfb, d0, nft, d1;
  block_exscan2(nf, 0, nfb, d0, nft, d1, ms->wsum);
  const int64_t ncand = L - nft;
  const int keff = (int)std::min<int64_t>(k, ncand);
  if (keff > 0) {
    // 11-bit radix digits over the 64-bit keys (at most 6 passes), finished inside one warp as
    // soon as the boundary digit holds <= 32 keys
    constexpr int NB11 = 2048, UNR = 8;
    __shared__ int hist11[NB11];
    __shared__ uint64_t list64[32];
    __shared__ uint64_t kth_s;
    __shared__ int nlist;
    if (tid == 0) ms->rem_sel = keff;
    uint64_t prefix = 0;
    int hi = 64, need_eq = -1;
    while (hi > 0) {
      const int dbits = hi >= 11 ? 11 : hi;
      const int sh = hi - dbits;
      for (int i = tid; i < NB11; i += DT) hist11[i] = 0;
      if (tid == 0) nlist = 0;
      __syncthreads();
      const uint64_t want = hi >= 64 ? 0ull : (prefix >> hi);
      for (int64_t i0 = 0; i0 < L; i0 += (int64_t)DT * UNR) {
        uint64_t key[UNR];
        bool ok[UNR];
#pragma unroll
        for (int j = 0; j < UNR; ++j) {
          const int64_t i = i0 + (int64_t)j * DT + tid;
          ok[j] = i < L && !((forced[i >> 5] >> (i & 31)) & 1u);
          key[j] = ok[j] ? score_key(s, is_f32, i) : 0;
        }
#pragma unroll
        for (int j = 0; j < UNR; ++j)
          if (ok[j] && (hi >= 64 ? 0ull : (key[j] >> hi)) == want) atomicAdd(&hist11[(key[j] >> sh) & (NB11 - 1)], 1);
      }
      __syncthreads();
      pick_digit_big<Cta256, NB11>(hist11, ms);
      const int d = ms->digit, nb = hist11[d];
      const int rem = ms->rem_sel - ms->cnt_above;
      __syncthreads();                  // every read of ms precedes the update (racecheck-clean)
      prefix |= (uint64_t)d << sh;
      hi = sh;
      if (tid == 0) ms->rem_sel = rem;
      __syncthreads();
      if (hi > 0 && nb <= 32) {
        // exact rank among the boundary digit's few keys
        const uint64_t w2 = prefix >> hi;
        for (int64_t i = tid; i < L; i += DT) {
          if ((forced[i >> 5] >> (i & 31)) & 1u) continue;
          const uint64_t key = score_key(s, is_f32, i);
          if ((key >> hi) == w2) list64[atomicAdd(&nlist, 1)] = key;
        }
        __syncthreads();
        if (tid < 32) {
          const uint64_t v = tid < nb ? list64[tid] : 0ull;
          int gtc = 0, eqc = 0;
          for (int j = 0; j < nb; ++j) { gtc += list64[j] > v; eqc += list64[j] == v; }
          __syncwarp();
          if (tid < nb && gtc < rem && rem <= gtc + eqc) { kth_s = v; ms->digit = rem - gtc; }
        }
        __syncthreads();
        prefix = kth_s;
        need_eq = ms->digit;
        __syncthreads();
        break;
      }
    }
    if (need_eq < 0) need_eq = ms->rem_sel;
    for (int64_t i = tid; i < L; i += DT) {
      if ((forced[i >> 5] >> (i & 31)) & 1u) continue;
      const uint64_t key = score_key(s, is_f32, i);
      if (key > prefix) atomicOr(&gt[i >> 5], 1u << (i & 31));
      else if (key == prefix) atomicOr(&eq[i >> 5], 1u << (i & 31));
    }
    __syncthreads();
    // keep the lowest-index need_eq of the ties
    const int per = (W + DT - 1) / DT;
    const int w0 = tid * per, w1 = std::min(W, w0 + per);
    int my = 0;
    for (int x = w0; x < w1; ++x) my += __popc(eq[x]);
    int before, dd, tt, t2;
    block_exscan2(my, 0, before, dd, tt, t2, ms->wsum);
    for (int x = w0; x < w1; ++x) {
      uint32_t e = eq[x];
      const int take = std::min(std::max(need_eq - before, 0), __popc(e));
      before += __popc(e);
      while (__popc(e) > take) e &= ~(1u << (31 - __clz(e)));
      gt[x] |= e;
    }
    __syncthreads();
  }
  // ordered emission
  const int per = (W + DT - 1) / DT;
  const int w0 = tid * per, w1 = std::min(W, w0 + per);
  int n = 0;
  for (int x = w0; x < w1; ++x) n += __popc(gt[x] | forced[x]);
  int pos, dd, tot, t2;
  block_exscan2(n, 0, pos, dd, tot, t2, ms->wsum);
  for (int x = w0; x < w1; ++x) {
    uint32_t b = gt[x] | forced[x];
    while (b) { const int i = __ffs(b) - 1; b &= b - 1; out[u * out_stride + pos++] = x * 32 + i; }
  }
  if (tid == 0) { counts[2 * u] = tot; counts[2 * u + 1] = keff; }
}

// ---------------------------------------------------------------- row dequantisation
__device__ __forceinline__ double deq_elem(const uint8_t* pay, const __half* sc, const __half* zp,
                                           int64_t row, int d, const RefPlanes& p) {
  const int c = (pay[row * p.payb + (d >> p.lper)] >> ((d & ((1 << p.lper) - 1)) << p.lbits)) & ((1 << p.bits) - 1);
  const int64_t pi = row * p.ngroups + (d >> p.lgs);
  return __dadd_rn(__dmul_rn((double)c, (double)__half2float(sc[pi])), (double)__half2float(zp[pi]));
}

// K'[row][d] of a dynamic (non-forced) token
__device__ __forceinline__ double key_elem(const RefPlanes& p, int64_t u, int64_t t, int d) {
  const int64_t row = u * p.L + t;
  if (p.bits == 16) return p.kfull[row * p.D + d];
  if (!p.siq) return deq_elem(p.kq, p.ks, p.kz, row, d, p);
  const int G = p.D / 4, rowb = (G + 1) / 2;
  const int g = d >> 2, i = d & 3;
  const int code = (p.codes[row * rowb + (g >> 1)] >> (4 * (g & 1))) & 15;
  const double sg = ((code >> (3 - i)) & 1) ? 1.0 : -1.0;
  const double m = deq_elem(p.kq, p.ks, p.kz, row, d, p);
  return __dmul_rn(__dmul_rn(sg, p.alpha[u * p.D + d]), m);
}
__device__ __forceinline__ double value_elem(const RefPlanes& p, int64_t u, int64_t t, int d) {
  const int64_t row = u * p.L + t;
  if (p.bits == 16) return p.vfull[row * p.D + d];
  return deq_elem(p.vq, p.vs, p.vz, row, d, p);
}

// which = 0 values, 1 keys (cache.gather semantics for dynamic rows)
__global__ void dequant_rows_kernel(RefPlanes p, const int64_t* __restrict__ rows, int64_t n, int which,
                                    double* __restrict__ out) {
  const int64_t u = blockIdx.y;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int d = threadIdx.x; d < p.D; d += blockDim.x) {
      const int64_t t = rows[i];
      out[(u * n + i) * p.D + d] = which ? key_elem(p, u, t, d) : value_elem(p, u, t, d);
    }
}

// ---------------------------------------------------------------- sparse attention, float64
// One CTA per (unit, query head).  Row sources follow cache.gather (cache.py:118-158).
__device__ __forceinline__ const double* forced_row(const AttendArgs& a, int64_t u, int64_t t, bool key) {
  if (t >= a.p.L) return (key ? a.rec_k : a.rec_v) + (u * a.rcap + (t - a.p.L)) * a.p.D;
  int lo = 0, hi = a.S - 1;
  const int32_t* si = a.sink_idx + u * a.S;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (si[mid] == t) return (key ? a.sink_k : a.sink_v) + (u * a.S + mid) * a.p.D;
    if (si[mid] < t) lo = mid + 1; else hi = mid - 1;
  }
  return nullptr;
}

// ATT_SPLIT CTAs per (unit, head), CTA z taking the selected rows [z n / S, (z + 1) n / S):
// a warp per row (32 warps, two rows in flight each; the rows are scattered over HBM), the
// row's source resolved once (cache.gather), each lane owning channels lane + 32 j; logits by a
// lane sum + warp tree (float64); the CTA's (max, sum, P V) written as a partial, and the last
// CTA of the (unit, head) (a counter the launcher zeroes) merges the partials in CTA order.
// Every order is fixed (deterministic); it differs from numpy's only by float64 rounding.
constexpr int ATT_NT = 1024;
constexpr int ATT_MAXD = 128;                 // channels: ATT_MAXD / 32 per lane
__global__ void __launch_bounds__(ATT_NT) attend_f64_kernel(AttendArgs a) {
  constexpr int NW = ATT_NT / 32, PER = ATT_MAXD / 32;
  __shared__ double red[NW];
  __shared__ double part[NW][ATT_MAXD];
  __shared__ int last;
  const int64_t u = blockIdx.x;
  const int h = blockIdx.y, z = blockIdx.z, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, D = a.p.D;
  const int64_t uh = u * a.H + h;
  const int n = a.nsel[u];
  const int i_lo = (int)((int64_t)z * n / ATT_SPLIT), i_hi = (int)((int64_t)(z + 1) * n / ATT_SPLIT);
  const int32_t* sel = a.sel + u * a.sel_stride;
  const double* q = a.q + uh * D;
  double* lg = a.ws + uh * (int64_t)a.sel_stride;
  const double scale = sqrt((double)D);
  double qv[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) qv[j] = 32 * j + lane < D ? q[32 * j + lane] : 0.0;
  double mx = -INFINITY;
  for (int i0 = i_lo + warp; i0 < i_hi; i0 += 2 * NW) {
    double s[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = i0 + r * NW;
      if (i >= i_hi) continue;
      const int64_t t = sel[i];
      const double* fr = forced_row(a, u, t, true);
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int d = 32 * j + lane;
        if (d < D) s[r] = __fma_rn(fr ? fr[d] : key_elem(a.p, u, t, d), qv[j], s[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o);
      const int i = i0 + r * NW;
      if (i < i_hi) {
        const double v = s[r] / scale;
        if (lane == 0) lg[i] = v;
        mx = fmax(mx, v);
      }
    }
  }
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < NW; ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  double sum = 0.0;
  for (int i = i_lo + tid; i < i_hi; i += ATT_NT) {
    const double w = exp(lg[i] - mx);
    lg[i] = w;
    sum += w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  double csum = 0.0;
  for (int w = 0; w < NW; ++w) csum += red[w];
  double acc[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) acc[j] = 0.0;
  for (int i0 = i_lo + warp; i0 < i_hi; i0 += 2 * NW) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = i0 + r * NW;
      if (i >= i_hi) continue;
      const int64_t t = sel[i];
      const double* fr = forced_row(a, u, t, false);
      const double w = lg[i];
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int d = 32 * j + lane;
        if (d < D) acc[j] = __fma_rn(w, fr ? fr[d] : value_elem(a.p, u, t, d), acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (32 * j + lane < D) part[warp][32 * j + lane] = acc[j];
  __syncthreads();
  // this CTA's partial: [max, sum, P V [D]]
  double* pz = a.part + (uh * ATT_SPLIT + z) * (ATT_MAXD + 2);
  for (int d = tid; d < D; d += ATT_NT) {
    double o = part[0][d];
    for (int w = 1; w < NW; ++w) o += part[w][d];
    pz[2 + d] = o;
  }
  if (tid == 0) { pz[0] = mx; pz[1] = csum; }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(a.cnt + uh, 1u) == ATT_SPLIT - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double* p0 = a.part + uh * ATT_SPLIT * (ATT_MAXD + 2);
  double M = -INFINITY;
  for (int zz = 0; zz < ATT_SPLIT; ++zz) M = fmax(M, __ldcg(p0 + zz * (ATT_MAXD + 2)));
  double tot = 0.0;
  for (int zz = 0; zz < ATT_SPLIT; ++zz) {
    const double mz = __ldcg(p0 + zz * (ATT_MAXD + 2));
    if (mz != -INFINITY) tot += __ldcg(p0 + zz * (ATT_MAXD + 2) + 1) * exp(mz - M);
  }
  for (int d = tid; d < D; d += ATT_NT) {
    double o = 0.0;
    for (int zz = 0; zz < ATT_SPLIT; ++zz) {
      const double mz = __ldcg(p0 + zz * (ATT_MAXD + 2));
      if (mz != -INFINITY) o += __ldcg(p0 + zz * (ATT_MAXD + 2) + 2 + d) * exp(mz - M);
    }
    a.out[uh * D + d] = o / tot;
  }
  if (tid == 0 && a.chk) {            // the weights' sum: sum_z sum_z e^(m_z - M) / tot
    double c = 0.0;
    for (int zz = 0; zz < ATT_SPLIT; ++zz) {
      const double mz = __ldcg(p0 + zz * (ATT_MAXD + 2));
      if (mz != -INFINITY) c += __ldcg(p0 + zz * (ATT_MAXD + 2) + 1) * exp(mz - M) / tot;
    }
    a.chk[uh] = c;
  }
}




// ---------------------------------------------------------------- elementwise helpers
// out[u][t][d] = x[u][t][d] - mu[u][d]  (apply_normalization, normalize.py:64-69)
__global__ void center_kernel(const void* __restrict__ x, int dt, int64_t L, int D, const double* __restrict__ mu,
                              double* __restrict__ out) {
  const int64_t u = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L * D; i += (int64_t)gridDim.x * blockDim.x)
    out[u * L * D + i] = __dsub_rn(load_in(x, dt, u * L * D + i), mu[u * D + i % D]);
}

// ---------------------------------------------------------------- host launchers
cudaError_t launch_lut_f64(const double* q, const double* cent, int64_t U, int G, int sign_only, double* out,
                           cudaStream_t st) {
  lut_f64_kernel<<<(unsigned)U, 256, 0, st>>>(q, cent, G, sign_only, out);
  return cudaGetLastError();
}

cudaError_t launch_score_f64(const double* lut, const uint8_t* codes, int64_t U, int G, int64_t L, double* out,
                             cudaStream_t st) {
  const int bx = (int)std::min<int64_t>(1024, (L + 127) / 128);
  score_f64_kernel<<<dim3(bx, (unsigned)U), 128, G * 16 * sizeof(double), st>>>(lut, codes, G, L, out);
  return cudaGetLastError();
}

size_t topk_workspace_bytes(int64_t U, int64_t L) { return (size_t)U * 3 * ((L + 31) / 32) * 4; }

cudaError_t launch_topk(const void* scores, int is_f32, int64_t U, int64_t L, const int32_t* forced, int F, int k,
                        void* ws, int32_t* out, int out_stride, int32_t* counts, cudaStream_t st) {
  topk_kernel<<<(unsigned)U, DT, 0, st>>>(scores, is_f32, L, forced, F, k, (uint32_t*)ws, out, out_stride, counts);
  return cudaGetLastError();
}

cudaError_t launch_dequant_rows(const RefPlanes& p, int64_t U, const int64_t* rows, int64_t n, int which,
                                double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int bx = (int)std::min<int64_t>(n, 4096);
  dequant_rows_kernel<<<dim3(bx, (unsigned)U), 128, 0, st>>>(p, rows, n, which, out);
  return cudaGetLastError();
}

cudaError_t launch_attend_f64(const AttendArgs& a, int64_t U, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.cnt, 0, (size_t)U * a.H * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  attend_f64_kernel<<<dim3((unsigned)U, a.H, ATT_SPLIT), ATT_NT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_center(const void* x, int dt, int64_t U, int64_t L, int D, const double* mu, double* out,
                          cudaStream_t st) {
  const int bx = (int)std::min<int64_t>(4096, (L * D + 255) / 256);
  center_kernel<<<dim3(bx, (unsigned)U), 256, 0, st>>>(x, dt, L, D, mu, out);
  return cudaGetLastError();
}

}  // namespace sikv
