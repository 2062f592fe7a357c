// Split-unit decode (sm_100a): one thread-block CLUSTER of NS CTAs per decode unit, for
// long contexts with few units (C3: 128K tokens, batch 1; head-sharded C3 leaves only
// 32-128 units per GPU).  CTA r of the cluster owns the token slice
// [r * nchunks / NS, (r+1) * nchunks / NS) of 256-token chunks and runs the phases of
// decode_step_kernel on it; the unit-wide decisions go through distributed shared memory:
//
//   threshold   sample counts / extremes and the 256-bin sample histogram are summed over
//               the cluster, so every CTA derives the same tau (and the same retries)
//   k-th key    each radix pass sums the CTAs' 4096-bin histograms in place
//   ties        CTA r keeps the key == K* ties left after CTAs 0..r-1 (lowest index first)
//   selection   CTA r writes its sorted slice at the prefix of the lower CTAs' counts
//   attention   every CTA attends its own selected rows (CTA 0 also the sinks / recents);
//               the (max, denominator, numerator) partials are combined in rank order
//
// Selections are identical to decode_step_kernel's (same keys, same rule); outputs match
// within float32 rounding of the different partial grouping.
#include "common.cuh"
#include "select.cuh"
#include "decode_common.cuh"
#include "api_types.cuh"
#include <cooperative_groups.h>
#include <math.h>
#include <algorithm>

namespace cg = cooperative_groups;

namespace sikv {

struct XSlot {                       // per-CTA exchange words (read remotely)
  int nsv;
  uint32_t kmx, kmn;
  int total, maxwc, bad;
  uint32_t maxx;
  int eqc, nsl;
};

struct ClusterX {
  static constexpr bool kCluster = true;
  int ns;
  XSlot* slot;
  __device__ __forceinline__ static void csync() { cg::this_cluster().sync(); }
  template <typename T>
  __device__ __forceinline__ static T* at(T* p, int r) { return cg::this_cluster().map_shared_rank(p, r); }

  __device__ __forceinline__ void sample(int& nsv, uint32_t& kmx, uint32_t& kmn) const {
    if (threadIdx.x == 0) { slot->nsv = nsv; slot->kmx = kmx; slot->kmn = kmn; }
    csync();
    nsv = 0; kmx = 0; kmn = 0xFFFFFFFFu;
    for (int r = 0; r < ns; ++r) {
      const XSlot* s = at(slot, r);
      nsv += s->nsv; kmx = max(kmx, s->kmx); kmn = min(kmn, s->kmn);
    }
    csync();
  }
  __device__ __forceinline__ void hist256(const int*& th, const uint32_t*& tmin) const {
    int* h = const_cast<int*>(th);
    uint32_t* m = const_cast<uint32_t*>(tmin);
    csync();
    int v = 0;
    uint32_t mv = 0xFFFFFFFFu;
    if (threadIdx.x < 256)
      for (int r = 0; r < ns; ++r) { v += at(h, r)[threadIdx.x]; mv = min(mv, at(m, r)[threadIdx.x]); }
    csync();
    if (threadIdx.x < 256) { h[threadIdx.x] = v; m[threadIdx.x] = mv; }
    __syncthreads();
  }
  __device__ __forceinline__ void counts(int& total, int& maxwc, bool& bad) const {
    if (threadIdx.x == 0) { slot->total = total; slot->maxwc = maxwc; slot->bad = bad ? 1 : 0; }
    csync();
    total = 0; maxwc = 0; bad = false;
    for (int r = 0; r < ns; ++r) {
      const XSlot* s = at(slot, r);
      total += s->total; maxwc = max(maxwc, s->maxwc); bad |= s->bad != 0;
    }
    csync();
  }
  template <int NBINT = NBIN>
  __device__ __forceinline__ const int* hist4k(const int* hc) const {
    int* h = const_cast<int*>(hc);
    constexpr int PER = NBINT / DT;
    int v[PER];
    csync();
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = 0;
    for (int r = 0; r < ns; ++r) {
      const int* hr = at(h, r);
#pragma unroll
      for (int j = 0; j < PER; ++j) v[j] += hr[threadIdx.x + DT * j];
    }
    csync();
#pragma unroll
    for (int j = 0; j < PER; ++j) h[threadIdx.x + DT * j] = v[j];
    __syncthreads();
    return h;
  }
  __device__ __forceinline__ uint32_t maxu(uint32_t x) const {
    if (threadIdx.x == 0) slot->maxx = x;
    csync();
    uint32_t m = 0;
    for (int r = 0; r < ns; ++r) m = max(m, at(slot, r)->maxx);
    csync();
    return m;
  }
};

__device__ long long* g_prof_split = nullptr;   // optional per-unit phase clocks of cluster rank 0
cudaError_t set_decode_split_profile(long long* p) { return cudaMemcpyToSymbol(g_prof_split, &p, sizeof(p)); }
#define SPROF(i) do { if (prof && tid == 0) prof[i] = clock64(); } while (0)

constexpr int SPLIT_NBIN = 512;

struct SplitArgs {
  const uint8_t* signs; const uint8_t* recs; const float* cent32; const float* alpha32;
  const int32_t* sink_idx; const uint32_t* ffrag; const int32_t* rn; const int32_t* umap; const float* q;
  float* out; float* lse; int32_t* sel; int32_t* sel_count; int32_t* diag;
  int64_t L;
  int fblocks, S, R, Gq, k, capw, sel_stride, ns, wmax;
  int lut_mode;                 // 0: centroid LUT, 1: sign-only LUT
  int off_cand, off_forced, off_misc, off_dyn, off_hist, off_bits, off_stage, off_x;
};

__global__ void __launch_bounds__(DT, 2) decode_split_kernel(SplitArgs a) {
  extern __shared__ __align__(128) char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ns = a.ns;
  const int rank = (int)cg::this_cluster().block_rank();
  const int64_t u = blockIdx.x / ns;
  const int64_t cu = a.umap ? (int64_t)a.umap[u] : u;            // the unit's cache
  const int64_t Lu = a.L;
  const int S = a.S, Gq = a.Gq;
  const int Ru = a.rn ? a.rn[cu] : a.R;   // recent rows of this unit
  // ---------------- this CTA's slice of the unit
  const int nch = (int)((Lu + 255) >> 8);
  const int c_lo = (int)((int64_t)rank * nch / ns), c_hi = (int)((int64_t)(rank + 1) * nch / ns);
  const int64_t t_lo = (int64_t)c_lo * 256, t_hi = min(Lu, (int64_t)c_hi * 256);
  const int64_t Ls = t_hi > t_lo ? t_hi - t_lo : 0;
  const int W = (int)((Ls + 31) >> 5);

  long long* prof = g_prof_split && rank == 0 ? g_prof_split + u * 16 : nullptr;
  SPROF(0);
  char* T = sm;                                                    // pair table while scoring
  uint32_t* cand = reinterpret_cast<uint32_t*>(sm + a.off_cand);
  uint32_t* forced = reinterpret_cast<uint32_t*>(sm + a.off_forced);
  Misc* ms = reinterpret_cast<Misc*>(sm + a.off_misc);
  XSlot* slot = reinterpret_cast<XSlot*>(sm + a.off_misc + 192);
  float* qs = reinterpret_cast<float*>(sm + a.off_misc + 256);     // [Gq][128]
  float* lut = qs + 8 * FD;
  float* qbar = lut + 512;
  float* inva = qbar + FD;
  float* ahat = inva + FD;
  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + (cu * Lu + t_lo) * FSIGN);
  const int32_t* sidx = a.sink_idx + cu * S;
  ClusterX xch{ns, slot};

  // geometry of the slice; the selection parameters are the unit's
  UnitGeom g;
  g.L = Ls;
  g.S = S;
  g.ncand = Lu - S;
  g.keff = (int)((int64_t)a.k < g.ncand ? (int64_t)a.k : g.ncand);
  g.nchunks = c_hi - c_lo;
  g.capw = a.capw;
  g.mode = g.keff == 0 ? 0 : (g.keff == g.ncand ? 1 : 3);
  g.sstride = g.mode == 3 ? (max(16, (g.nchunks + MAX_SAMPLE_CHUNKS - 1) / MAX_SAMPLE_CHUNKS) + NB - 1) / NB * NB : 1;
  g.nsc = g.mode == 3 ? (g.nchunks + g.sstride - 1) / g.sstride : 0;
  g.npass = 1;                       // the cluster merges one register-resident sample pass
  {
    int64_t f = S > 0 ? (int64_t)sidx[S - 1] + 1 - t_lo : 0;
    f = f < 0 ? 0 : (f > Ls ? Ls : f);
    g.flim = f;
  }
  uint4 wsamp[MAX_SAMPLE_CHUNKS];
  load_sample(g, signs, tid, wsamp);

  // ---------------- A: queries, LUT, pair table, forced bitmap of the slice
  for (int i = tid; i < Gq * FD; i += DT) qs[i] = a.q[u * Gq * FD + i];
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  if (tid == 0) ms->fb = 0;
  __syncthreads();
  for (int j = tid; j < S; j += DT) {
    const int64_t t = sidx[j] - t_lo;
    if (t >= 0 && t < Ls) atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  if (tid < FD) {
    float s = qs[tid];
    for (int h = 1; h < Gq; ++h) s = __fadd_rn(s, qs[h * FD + tid]);
    qbar[tid] = s;
    const float al = a.alpha32[cu * FD + tid];
    ahat[tid] = al > 0.f ? al : 1.0f;
    inva[tid] = 1.0f / ahat[tid];
  }
  __syncthreads();
  build_pair_table<Cta256>(a.cent32 + cu * 32 * 16 * 4, qbar, lut, T, a.lut_mode);
  SPROF(1);

  // ---------------- B/C: candidates, the unit's k-th key, bitmaps of the slice
  const int mode = g.mode;
  uint32_t* gt = reinterpret_cast<uint32_t*>(sm + a.off_bits);
  uint32_t* eq = gt + a.wmax;
  uint32_t kstar = 0;
  int need_eq = 0, eq_count = 0;
  if (mode >= 2) {
    uint32_t tau;
    const bool fb = produce_candidates<Cta256, ClusterX>(g, signs, T, forced, wsamp, cand,
                                                         reinterpret_cast<int*>(cand), cand + 256, ms, tau, xch);
    SPROF(2);
    if (!fb) {
      // 512-bin radix passes: each pass sums ns x 2 KB of histograms over the cluster (with
      // 2048 bins the distributed-shared-memory merge was a third of the kernel at 8 CTAs)
      select_from_candidates<Cta256, ClusterX, SPLIT_NBIN>(g, cand, ms->wcnt, ms->maxx, tau,
                                               reinterpret_cast<int*>(sm + a.off_hist), ms, gt, eq, kstar,
                                               need_eq, eq_count, xch);
    } else {
      if (tid == 0) ms->fb = 1;
      gt = cand + NBIN + 64;                                       // candidates are void
      eq = gt + a.wmax;
      produce_exact<Cta256, ClusterX>(g, signs, T, forced, reinterpret_cast<int*>(cand), ms, gt, eq, kstar,
                                      need_eq, eq_count, xch);
    }
  }
  SPROF(3);
  // ties: the lower ranks (lower token indices) take theirs first
  if (tid == 0) slot->eqc = eq_count;
  ClusterX::csync();
  int eq_before_rank = 0;
  for (int r = 0; r < rank; ++r) eq_before_rank += ClusterX::at(slot, r)->eqc;
  ClusterX::csync();
  const int take = mode >= 2 ? min(max(need_eq - eq_before_rank, 0), eq_count) : 0;

  // ---------------- ordered emission of the slice
  int32_t* dyn = reinterpret_cast<int32_t*>(sm + a.off_dyn);
  int ndyn;
  {
    const int per = (W + DT - 1) / DT;
    const int w0 = min(W, tid * per), w1 = min(W, w0 + per);
    const bool all_eq = mode < 2 || eq_count == take;
    int eq_before = 0;
    if (!all_eq) {
      int my_eq = 0;
      for (int x = w0; x < w1; ++x) my_eq += __popc(eq[x]);
      int dummy, t1, t2;
      block_exscan2<Cta256>(my_eq, 0, eq_before, dummy, t1, t2, ms->wsum);
    }
    auto dbits = [&](int x, int& eb) -> uint32_t {
      if (mode == 0) return 0u;
      if (mode == 1) {
        uint32_t d = ~forced[x];
        if (x == W - 1 && (Ls & 31)) d &= (1u << (Ls & 31)) - 1u;
        return d;
      }
      uint32_t e = eq[x];
      if (!all_eq) {
        const int tk = min(max(take - eb, 0), __popc(e));
        eb += __popc(e);
        while (__popc(e) > tk) e &= ~(1u << (31 - __clz(e)));
      }
      return gt[x] | e;
    };
    int nd = 0, nsl = 0, eb = eq_before;
    for (int x = w0; x < w1; ++x) {
      const uint32_t d = dbits(x, eb);
      nd += __popc(d);
      nsl += __popc(d | forced[x]);
    }
    int dpos, spos, dtot, stot;
    block_exscan2<Cta256>(nd, nsl, dpos, spos, dtot, stot, ms->wsum);
    pad_dyn(dyn, dtot, tid);
    if (tid == 0) slot->nsl = stot;
    ClusterX::csync();
    int soff = 0, sall = 0;
    for (int r = 0; r < ns; ++r) {
      const int c = ClusterX::at(slot, r)->nsl;
      if (r < rank) soff += c;
      sall += c;
    }
    int32_t* sel_u = a.sel ? a.sel + u * a.sel_stride : nullptr;
    eb = eq_before;
    for (int x = w0; x < w1; ++x) {
      uint32_t d = dbits(x, eb);
      uint32_t sb = d | forced[x];
      const int32_t base = (int32_t)(t_lo + 32 * x);
      while (d) { const int b = __ffs(d) - 1; d &= d - 1; dyn[dpos++] = base + b; }
      if (sel_u)
        while (sb) { const int b = __ffs(sb) - 1; sb &= sb - 1; sel_u[soff + spos++] = base + b; }
    }
    if (rank == ns - 1) {
      if (sel_u)
        for (int r = tid; r < Ru; r += DT) sel_u[sall + r] = (int32_t)(Lu + r);
      if (tid == 0 && a.sel_count) a.sel_count[u] = sall + Ru;
    }
    if (tid == 0 && rank == 0 && a.diag) a.diag[u] = (mode & 3) | (ms->fb ? 4 : 0) | 8;
    __syncthreads();
    ndyn = dtot;
  }

  SPROF(4);
  // ---------------- D: sparse attention over this slice's rows (+ forced rows on rank 0)
  Attn A;
  attn_init(A, qs, ahat, Gq, lane);
  const int nf = rank == 0 ? S + Ru : 0;
  const int nbf = (nf + 15) >> 4;
  if (nf > 0) attn_forced(A, a.ffrag + cu * a.fblocks * FBLK_WORDS, nf, warp, DW, lane);
  attn_dynamic(A, a.recs + cu * Lu * FREC, dyn, ndyn, (warp - nbf % DW + DW) % DW, DW,
               sm + a.off_stage + warp * 2 * STAGE_BYTES, lane);
  __syncthreads();
  // this CTA's (max, denominator, unnormalised numerator) per head, warps combined in order
  float* part = reinterpret_cast<float*>(sm + a.off_stage);        // [DW][Gq][128] (staging is dead)
  float* pm = part + DW * Gq * FD;
  float* pl = pm + DW * Gq;
  float* xnum = reinterpret_cast<float*>(sm + a.off_x);           // [Gq][128]
  float* xm = xnum + Gq * FD;                                      // [Gq]
  float* xden = xm + 8;                                            // [Gq]
  SPROF(5);
  attn_write_partial(A, part, pm, pl, warp, Gq, lane);
  __syncthreads();
  for (int e = tid; e < Gq * FD; e += DT) {
    const int h = e / FD, d = e % FD;
    float M = -INFINITY;
    for (int w = 0; w < DW; ++w) M = fmaxf(M, pm[w * Gq + h]);
    float num = 0.f, den = 0.f;
    for (int w = 0; w < DW; ++w) {
      const float mw = pm[w * Gq + h];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      num += part[(w * Gq + h) * FD + d] * f;
      den += pl[w * Gq + h] * f;
    }
    xnum[e] = num;
    if (d == 0) { xm[h] = M; xden[h] = den; }
  }
  ClusterX::csync();
  // rank-ordered combine; CTA r finalises elements r, r + ns, ...
  for (int e = rank + ns * tid; e < Gq * FD; e += ns * DT) {
    const int h = e / FD, d = e % FD;
    float M = -INFINITY;
    for (int r = 0; r < ns; ++r) M = fmaxf(M, ClusterX::at(xm, r)[h]);
    float num = 0.f, den = 0.f;
    for (int r = 0; r < ns; ++r) {
      const float mr = ClusterX::at(xm, r)[h];
      const float f = mr == -INFINITY ? 0.f : exp2f(mr - M);
      num += ClusterX::at(xnum, r)[e] * f;
      den += ClusterX::at(xden, r)[h] * f;
    }
    a.out[(u * Gq) * FD + e] = num / den;
    if (a.lse && d == 0) a.lse[u * Gq + h] = (M + log2f(den)) * 0.6931471805599453f;
  }
  ClusterX::csync();                 // remote reads of this CTA's shared memory are done
  SPROF(6);
}

// ---------------------------------------------------------------- host side
static int a128(int x) { return (x + 127) & ~127; }

struct SplitLayout { SplitArgs a; int total; };

static SplitLayout split_layout(int64_t L, int k, int S, int Gq, int cap, int ns) {
  SplitLayout r{};
  SplitArgs& a = r.a;
  const int nch = (int)((L + 255) / 256);
  const int maxch = (nch + ns - 1) / ns;
  const int64_t Ls = std::min<int64_t>(L, (int64_t)maxch * 256);
  const int W = (int)((Ls + 31) / 32);
  const int keff = (int)std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  a.wmax = W;
  a.capw = std::max(32, cap / DW);
  // R0: pair table while scoring; then dyn | {hist, gt, eq} | later staging / partials
  a.off_dyn = 0;
  int u0 = a128((std::max(keff, 1) + 16) * 4);
  a.off_hist = u0;
  a.off_bits = a128(u0 + (NBIN + 64) * 4);
  const int sel_end = a.off_bits + 2 * W * 4;
  a.off_stage = u0;
  const int att_end = u0 + std::max(DW * 2 * STAGE_BYTES, DW * Gq * (FD + 2) * 4);
  const int r0 = std::max(TBL_BYTES, a128(std::max(sel_end, att_end)));
  // R1: candidate segments; the sample histogram; the exact fallback's histogram + bitmaps
  int r1 = DW * a.capw * 8;
  r1 = std::max(r1, (NBIN + 64) * 4 + 2 * W * 4);
  r1 = std::max(r1, 512 * 4);
  a.off_cand = r0;
  int off = a.off_cand + a128(r1);
  a.off_forced = off;
  off += a128(W * 4);
  a.off_x = off;
  off += a128((8 * FD + 16) * 4);
  a.off_misc = off;
  off += 256 + (8 * FD + 512 + FD * 3) * 4;
  r.total = a128(off);
  return r;
}

int split_smem_bytes(int64_t L, int k, int S, int Gq, int cap, int ns) {
  return split_layout(L, k, S, Gq, cap, ns).total;
}

// candidate buffer per CTA: about twice the CTA's share of k, plus slack
int split_default_cap(int64_t L, int k, int S, int ns) {
  const int64_t keff = std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  return (int)std::max<int64_t>(1024, ((2 * keff / ns + 1024) + 63) / 64 * 64);
}

cudaError_t launch_decode_split(const uint8_t* signs, const uint8_t* recs, const float* cent32,
                                const float* alpha32, const int32_t* sink_idx, int S, const uint32_t* ffrag,
                                int fblocks, const int32_t* rn, int R, const float* q, int64_t U, int64_t L, int Gq, int k, int cap,
                                int ns, float* out, float* lse, int32_t* sel, int sel_stride, int32_t* sel_count,
                                int32_t* diag, const int32_t* umap, int lut_mode, cudaStream_t st) {
  SplitLayout lay = split_layout(L, k, S, Gq, cap, ns);
  SplitArgs a = lay.a;
  a.signs = signs; a.recs = recs; a.cent32 = cent32; a.alpha32 = alpha32; a.sink_idx = sink_idx; a.ffrag = ffrag; a.rn = rn; a.umap = umap;
  a.q = q; a.out = out; a.lse = lse; a.sel = sel; a.sel_count = sel_count; a.diag = diag;
  a.L = L; a.fblocks = fblocks; a.S = S; a.R = R; a.Gq = Gq; a.k = k; a.sel_stride = sel_stride; a.ns = ns;
  a.lut_mode = lut_mode;
  cudaError_t e = cudaFuncSetAttribute(decode_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(U * ns));
  cfg.blockDim = dim3(DT);
  cfg.dynamicSmemBytes = (size_t)lay.total;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)ns;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_split_kernel, a);
}

}  // namespace sikv
