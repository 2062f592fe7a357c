// Two-kernel decode step (sm_100a): selection and attention in separate launches, each with
// the occupancy its phase wants.
//
//   decode_select_kernel   one 512-thread CTA per SM, persistent.  Two independent groups of
//                          8 warps (named barriers 1 and 2) each own a unit at a time
//                          (units b + (2 it + g) * grid): pair table, sign-plane scoring,
//                          sampled threshold, exact k-th key and the dynamic list, written to
//                          the workspace.  The groups' 32-column pair tables interleave in one
//                          64 KiB region (ColKey), so 16 warps stream sign planes per SM while
//                          either group sits in its latency-bound setup / selection steps.
//   decode_attend_kernel   one 128-thread CTA (4 warps) per unit, four per SM, launched as a
//                          programmatic dependent of the selection grid: the unit's forced rows,
//                          then (griddepcontrol.wait) its dynamic list, sparse flash-decode
//                          (decode_common.cuh), fixed-order merge of the 4 warp partials.
//
// The arithmetic is that of decode.cu (shared device code): selections are identical; the
// attention splits a unit over 4 warps instead of 8, so outputs agree with the one-CTA path to
// the fp16 rounding of P against each warp's running max (not bit for bit).
// Tried and removed: TMA tile::gather4 row staging (5% slower than cp.async),
// sample keys in shared memory, padding the selection kernel's shared memory.
#include "common.cuh"
#include "select.cuh"
#include "api_types.cuh"
#include "decode_common.cuh"
#include "../../include/sikv_b200.h"
#include <algorithm>
#include <type_traits>

namespace sikv {

constexpr int SEL_THREADS = 512;
__device__ long long* g_prof_two = nullptr;   // optional per-unit phase clocks (profiling)
// the selection groups' radix digit: 9 bits (512 bins) — at C4 (1.4 K candidates per unit)
// 2.5% faster than 11 bits, neutral at C2; path 1 keeps 11 bits (C3: 6 K candidates)
constexpr int SEL_NBIN = 512;
using SG0 = NamedGroup<1, 0>;
using SG1 = NamedGroup<2, 256>;

struct TwoArgs {
  const uint8_t* signs;
  const uint8_t* recs;
  const float* cent32;
  const float* alpha32;
  const int32_t* sink_idx;
  const uint32_t* ffrag;
  const int32_t* rn;    // [U] recent rows per unit, nullable (then R)
  const int32_t* umap;  // [U] cache unit of each query unit (per-q-head policy), nullable = identity
  const float* q;
  float* out;
  float* lse;
  int32_t* sel;
  int32_t* sel_count;
  int32_t* diag;
  int32_t* ndyn;        // [U]
  int32_t* dynl;        // [U][dstride]
  uint32_t* gbits;      // [U][2W] fallback / sorted-selection bitmaps
  uint32_t* gforced;    // [U][W] forced bitmaps when they do not fit shared memory (long units)
  float* spart;         // [U][nsplit][Gq][FD + 2] split-attention partials (num, M, den), nsplit > 1
  int32_t* scnt;        // [U] split CTAs done (zeroed by the selection kernel)
  int nsplit;           // attention CTAs per unit (few units: fill the SMs)
  int64_t L, U;
  int fblocks, S, R, Gq, k, capw, sel_stride, dstride;
  int lut_mode;         // 0: centroid LUT, 1: sign-only LUT
  // select-kernel shared-memory layout (per group: misc | hist | forced | cand)
  int g_bytes, g_hist, g_forced, g_cand, g_pre;   // g_forced < 0: forced bitmap in gforced
  sikv_exchange x;      // fused multi-GPU output exchange (x.npeers 0: off)
};

// The fused output exchange: unit u's float32 rows (just written by this CTA) go as bf16 to
// row gid[u] of every rank's model-layout buffer over NVLink; after a system-scope fence the
// CTA adds its Gq rows to every rank's arrival counter (sikv_exchange_wait acquires them).
__device__ __forceinline__ void push_unit(const sikv_exchange& x, const float* out, int64_t u, int Gq, int tid,
                                          int nt) {
  __syncthreads();                                   // the unit's rows are in global memory
  const int n2 = Gq * FD / 2;
  const float2* o = reinterpret_cast<const float2*>(out + u * Gq * FD);
  const int64_t base = (int64_t)__ldg(x.unit_gid + u) * n2;
  for (int i = tid; i < n2; i += nt) {
    const float2 v = o[i];
    const __nv_bfloat162 b = __floats2bfloat162_rn(v.x, v.y);
    for (int p = 0; p < x.npeers; ++p) reinterpret_cast<__nv_bfloat162*>(x.out[p])[base + i] = b;
  }
  // the CTA barrier orders every thread's stores before the releasing reductions, whose
  // system-scope release makes them visible to the peer before its counter moves
  __syncthreads();
  if (tid < x.npeers)
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(x.flag[tid]), "l"((unsigned long long)Gq)
                 : "memory");
}

// the exchange for the paths whose kernels have no epilogue hook: one CTA per unit, after them
__global__ void __launch_bounds__(128) push_outputs_kernel(const sikv_exchange x, const float* __restrict__ out,
                                                           int Gq) {
  push_unit(x, out, blockIdx.x, Gq, threadIdx.x, 128);
}

cudaError_t launch_push_outputs(const sikv_exchange& x, const float* out, int64_t U, int Gq, cudaStream_t st) {
  push_outputs_kernel<<<(unsigned)U, 128, 0, st>>>(x, out, Gq);
  return cudaGetLastError();
}

// spins until every rank's rows of this step have arrived; a peer that never delivers (a rank
// died) traps after 20 s instead of hanging the stream
__global__ void exchange_wait_kernel(const unsigned long long* flag, unsigned long long target) {
  unsigned long long v, t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
}

cudaError_t launch_exchange_wait(const unsigned long long* flag, unsigned long long target, cudaStream_t st) {
  exchange_wait_kernel<<<1, 1, 0, st>>>(flag, target);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- selection
constexpr int SINK_STAGE = 256;   // sink indices staged with the next unit's inputs (more: read from L2)

// the group's staging area for the next unit's queries, centroids and sink indices (cp.async)
__device__ __forceinline__ void prefetch_unit(const TwoArgs& a, char* base, int tid, int64_t un) {
  const uint32_t pre_s = (uint32_t)__cvta_generic_to_shared(base + a.g_pre);
  if (un >= 0 && un < a.U) {
    for (int i = tid; i < a.Gq * FD / 4; i += DT)
      cp_async16_s(pre_s + 16u * (uint32_t)i, a.q + un * a.Gq * FD + 4 * i);
    const int64_t cn = a.umap ? (int64_t)__ldg(a.umap + un) : un;
    for (int i = tid; i < 512; i += DT)
      cp_async16_s(pre_s + (uint32_t)(a.Gq * FD * 4) + 16u * (uint32_t)i, a.cent32 + cn * 2048 + 4 * i);
    const uint32_t ps = pre_s + (uint32_t)((a.Gq * FD + 2048) * 4);
    for (int i = tid; i < min(a.S, SINK_STAGE); i += DT)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(ps + 4u * (uint32_t)i), "l"(a.sink_idx + cn * a.S + i));
  }
  cp_commit();
}

// one unit's selection by one 8-warp group: the unit's queries / centroids were prefetched
// into the staging area; `next` (or -1) is prefetched once they have been consumed.
// Returns the dynamic list length (the list is in a.dynl).
template <class PG, int G, bool XP>
__device__ __forceinline__ int select_unit(const TwoArgs& a, char* sm, int64_t u, int64_t next) {
  const int64_t L = a.L;
  const int W = (int)((L + 31) >> 5);
  const int S = a.S, Gq = a.Gq;
  const int tid = PG::tid();
  char* T = sm + 128 * G;                        // this group's columns of the shared table rows
  char* base = sm + TBL_BYTES + G * a.g_bytes;
  float* lut = reinterpret_cast<float*>(base);
  float* qbar = lut + 512;
  int* th = reinterpret_cast<int*>(qbar + FD);
  uint32_t* tmin = reinterpret_cast<uint32_t*>(th + 256);
  Misc* ms = reinterpret_cast<Misc*>(tmin + 256);
  int* hist = reinterpret_cast<int*>(base + a.g_hist);
  uint32_t* const forced_s = reinterpret_cast<uint32_t*>(base + (a.g_forced >= 0 ? a.g_forced : 0));
  uint32_t* cand = reinterpret_cast<uint32_t*>(base + a.g_cand);
  const float* pre_q = reinterpret_cast<const float*>(base + a.g_pre);   // [8][128]
  const float4* pre_c = reinterpret_cast<const float4*>(pre_q + Gq * FD);  // [512]
  long long* prof = g_prof_two ? g_prof_two + u * 16 : nullptr;
  if (prof && tid == 0) prof[0] = clock64();
  const int64_t cu = a.umap ? (int64_t)__ldg(a.umap + u) : u;    // the unit's cache
  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + cu * L * FSIGN);
  // the sample's loads first (its geometry does not depend on the sinks), the sink-dependent
  // limit once the staged sink indices are visible
  UnitGeom g = unit_geom(L, S, a.k, a.capw, nullptr, 0);
  uint4 wsamp[MAX_SAMPLE_CHUNKS];
  load_sample(g, signs, tid, wsamp);
  uint32_t* forced = a.g_forced >= 0 ? forced_s : a.gforced + u * W;
  const float* qs = pre_q;
  const int* sidx = S <= SINK_STAGE ? reinterpret_cast<const int*>(pre_q + Gq * FD + 2048) : a.sink_idx + cu * S;
  cp_wait<0>();                      // this unit's queries / centroids / sink indices have landed
  if (prof && tid == 0) prof[4] = clock64();
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  PG::sync();                        // (also makes every thread's staged data visible)
  g.flim = S > 0 ? (int64_t)sidx[S - 1] + 1 : 0;
  const int psid = tid < S ? sidx[tid] : -1;
  if (psid >= 0) atomicOr(&forced[psid >> 5], 1u << (psid & 31));
  for (int j = tid + DT; j < S; j += DT) {
    const int t = sidx[j];
    atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  if (tid < FD) {
    float sq = qs[tid];
    for (int h = 1; h < Gq; ++h) sq = __fadd_rn(sq, qs[h * FD + tid]);
    qbar[tid] = sq;
  }
  PG::sync();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = tid + DT * r, gg = e >> 4;
    const float4 c = lut_factors(pre_c[e], e & 15, a.lut_mode);
    const float q0 = qbar[4 * gg], q1 = qbar[4 * gg + 1], q2 = qbar[4 * gg + 2], q3 = qbar[4 * gg + 3];
    lut[(e & 15) * 32 + gg] = __fadd_rn(__fadd_rn(__fmul_rn(q0, c.x), __fmul_rn(q2, c.z)),
                                        __fadd_rn(__fmul_rn(q1, c.y), __fmul_rn(q3, c.w)));
  }
  PG::sync();                        // every read of the staged inputs is done
  if (prof && tid == 0) prof[5] = clock64();
  prefetch_unit(a, base, tid, next);
  build_pair_rows_col<PG>(lut, T);
  if (prof && tid == 0) prof[1] = clock64();
  const int mode = g.mode;
  int32_t* dyn = a.dynl + u * a.dstride;
  int32_t* sel_u = a.sel ? a.sel + u * a.sel_stride : nullptr;
  int32_t* sel_count_u = a.sel_count ? a.sel_count + u : nullptr;
  uint32_t* gt = a.gbits + u * 2 * W;
  uint32_t* eq = gt + W;
  int ndyn = -1, fb = 0, need_eq = 0, eq_count = 0;
  uint32_t kstar = 0;
  if (mode >= 2) {
    uint32_t tau;
    fb = produce_candidates<PG, NoX, ColKey, NB, XP>(g, signs, T, forced, wsamp, cand, th, tmin, ms, tau, NoX(), prof)
             ? 1 : 0;
    if (prof && tid == 0) prof[2] = clock64();
    if (!fb) {
      ndyn = select_emit_candidates<PG, SEL_NBIN>(g, forced, cand, ms->wcnt, ms->maxx, tau, hist, ms, gt, eq, dyn, sel_u,
                                        a.rn ? __ldg(a.rn + cu) : a.R, sel_count_u, kstar, prof);
    } else {
      produce_exact<PG, NoX, ColKey, SEL_NBIN>(g, signs, T, forced, hist, ms, gt, eq, kstar, need_eq, eq_count);
    }
  }
  if (ndyn < 0)
    ndyn = emit_selection<PG>(g, mode, forced, gt, eq, need_eq, eq_count, dyn, sel_u, a.rn ? __ldg(a.rn + cu) : a.R,
                              sel_count_u, ms);
  if (prof && tid == 0) prof[3] = clock64();
  if (tid == 0) {
    a.ndyn[u] = ndyn;
    if (a.nsplit > 1) a.scnt[u] = 0;
    if (a.diag) a.diag[u] = (mode & 3) | (fb ? 4 : 0);
  }
  PG::sync();                       // the group's shared memory is reused by its next unit
  return ndyn;
}

template <class PG, int G, bool XP>
__device__ __forceinline__ void select_group(const TwoArgs& a, char* sm) {
  prefetch_unit(a, sm + TBL_BYTES + G * a.g_bytes, PG::tid(), (int64_t)blockIdx.x + (int64_t)G * gridDim.x);
  for (int it = 0;; ++it) {
    const int64_t u = (int64_t)blockIdx.x + (int64_t)(2 * it + G) * gridDim.x;
    if (u >= a.U) break;
    select_unit<PG, G, XP>(a, sm, u, u + 2 * gridDim.x);
  }
}

// XP: long units (>= 64K tokens) with extra sample passes
template <bool XP>
__global__ void __launch_bounds__(SEL_THREADS, 1) decode_select_kernel(TwoArgs a) {
  extern __shared__ __align__(128) char sm[];
  // the attention grid may be scheduled onto SMs as this grid's CTAs retire: it attends the
  // forced rows, then waits for this grid to complete (griddepcontrol.wait) before the lists
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // group from a value the compiler can prove warp-uniform (uniform-datapath table base)
  const int grp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 8), 0);
  if (grp == 0) select_group<SG0, 0, XP>(a, sm);
  else select_group<SG1, 1, XP>(a, sm);
}

// ---------------------------------------------------------------- attention
// attention CTAs: NW warps each, 16 / NW per SM (16 warps per SM either way).  Units of at
// most ATT_SMALL_ROWS dynamic + forced rows take 2-warp CTAs when they fill at least two waves
// of them (C4, 7168 units: 0.743 -> 0.719 ms; 3584: 0.385 -> 0.378), else 4-warp CTAs (fewer,
// faster units: 1792 units 0.206 vs 0.213 ms, 896 units 0.118 vs 0.123; long units, C3: 0.205
// vs 0.215)
constexpr int ATT_WARPS_MAX = 4;
constexpr int ATT_SMALL_ROWS = 1536;
__host__ __device__ constexpr int att_ctas_per_sm(int nw) { return 16 / nw; }
static int att_warps(int64_t U, int64_t L, int k, int S, int nsm) {
  const int64_t keff = std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  return keff + S <= ATT_SMALL_ROWS && U >= 2LL * att_ctas_per_sm(2) * nsm ? 2 : 4;
}
constexpr int ATT_STAGES = 3;   // cp.async staging buffers per warp (2: C2 0.847 ms, 3: 0.843, 4: 0.847)

// One unit's attention by one CTA of NW warps.  Every warp starts on its own: q~ and the row
// indices come straight from global memory (L2), so the only CTA-wide barriers are the
// two around the partial merge.
// The unit's rows are dealt to the nsplit x NW warps of its CTAs (CTA part `sp`): with few
// units (C3) one CTA per unit would leave most warp slots idle.  Each CTA merges its warps;
// the last CTA of the unit to finish (counter) merges the CTA partials in split order, so
// the result does not depend on which CTA finishes last.
template <int NW, bool R16, bool SPLIT, bool XCH>
__device__ __forceinline__ void attend_unit(const TwoArgs& a, char* stage, int64_t u, int sp) {
  constexpr int NT = 32 * NW;
  const int tid = threadIdx.x, lane = tid & 31;
  const int nwa = SPLIT ? NW * a.nsplit : NW;      // warps attending the unit
  const int warp = sp * NW + (tid >> 5);           // this warp among them
  const int64_t cu = a.umap ? (int64_t)__ldg(a.umap + u) : u;    // the unit's cache
  const int S = a.S, R = a.rn ? __ldg(a.rn + cu) : a.R, Gq = a.Gq;
  const int32_t* dyn = a.dynl + u * a.dstride;
  const int nf = S + R;
  const int nbf = (nf + 15) >> 4;
  const uint32_t* ffrag_u = a.ffrag + cu * a.fblocks * FBLK_WORDS;
  // start the forced fragments and the list on their way to L2 while q~ loads
  for (int i = tid; i < (nbf * FBLK_WORDS * 4 + 127) / 128; i += NT)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(ffrag_u) + 128 * i));
  for (int i = tid; i < a.dstride / 32; i += NT)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(dyn) + 128 * i));
  const int lw = tid >> 5;
  Attn A;
  attn_init_g(A, a.q + u * Gq * FD, a.alpha32 + cu * FD, Gq, lane);
  attn_forced(A, ffrag_u, nf, warp, nwa, lane);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the selection grid is complete
  const int ndyn = __ldg(a.ndyn + u);
  if constexpr (R16)
    attn_dynamic16<ATT_STAGES>(A, a.recs + cu * a.L * FREC16, dyn, ndyn, (warp - nbf % nwa + nwa) % nwa, nwa,
                               stage + lw * ATT_STAGES * STAGE16_BYTES, lane);
  else
    attn_dynamic<ATT_STAGES>(A, a.recs + cu * a.L * FREC, dyn, ndyn, (warp - nbf % nwa + nwa) % nwa, nwa,
                             stage + lw * ATT_STAGES * STAGE_BYTES, lane);
  __syncthreads();
  float* part = reinterpret_cast<float*>(stage);
  float* pm = part + NW * Gq * FD;
  float* pl = pm + NW * Gq;
  attn_write_partial(A, part, pm, pl, lw, Gq, lane);
  __syncthreads();
  if constexpr (!SPLIT) {
    attn_merge<Cta256>(part, pm, pl, NW, Gq, tid, NT, a.out + u * Gq * FD, a.lse ? a.lse + u * Gq : nullptr);
  } else {
    // this CTA's partial (num, M, den per head) -> global; the last CTA merges
    float* sp_u = a.spart + u * a.nsplit * Gq * (FD + 2);
    attn_merge_partial(part, pm, pl, NW, Gq, tid, NT, sp_u + sp * Gq * (FD + 2));
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (tid == 0) last = atomicAdd(a.scnt + u, 1) == a.nsplit - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    attn_merge_splits(sp_u, a.nsplit, Gq, tid, NT, a.out + u * Gq * FD, a.lse ? a.lse + u * Gq : nullptr);
    if constexpr (XCH) push_unit(a.x, a.out, u, Gq, tid, NT);
  }
}

// R16: 16-bit records (512 B per token, stored fp16 fragments; 64 KB of staging per CTA);
// SPLIT: nsplit CTAs per unit; NW warps per CTA
// XCH: the fused output exchange epilogue (separate instances: its code perturbs the register
// allocation of the gather loop, +32 instructions per block, so the plain path never carries it)
template <bool R16, bool SPLIT, int NW, bool XCH = false>
__global__ void __launch_bounds__(32 * NW, 16 / NW) decode_attend_kernel(const __grid_constant__ TwoArgs a) {
  extern __shared__ __align__(128) char sm[];
  if constexpr (SPLIT) attend_unit<NW, R16, true, XCH>(a, sm, blockIdx.x / a.nsplit, (int)(blockIdx.x % a.nsplit));
  else {
    attend_unit<NW, R16, false, XCH>(a, sm, blockIdx.x, 0);
    if constexpr (XCH) push_unit(a.x, a.out, blockIdx.x, a.Gq, threadIdx.x, 32 * NW);
  }
}

// ---------------------------------------------------------------- host side
static int a128(int x) { return (x + 127) & ~127; }
cudaError_t set_decode_two_profile(long long* p) { return cudaMemcpyToSymbol(g_prof_two, &p, sizeof(p)); }

static int two_dstride(int64_t L, int k, int S) {
  const int keff = (int)std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  return (keff + 16 + 31) & ~31;
}

static TwoArgs two_layout(int64_t L, int k, int S, int cap, int Gq, bool forced_in_smem = true) {
  TwoArgs a{};
  const int W = (int)((L + 31) / 32);
  a.capw = std::max(32, cap / DW);
  int off = a128((512 + FD + 256 + 256) * 4 + (int)sizeof(Misc));
  a.g_hist = off;
  off += a128((SEL_NBIN + 64) * 4);
  a.g_forced = forced_in_smem ? off : -1;
  if (forced_in_smem) off += a128(W * 4);
  a.g_cand = off;
  off += a128(std::max(DW * a.capw * 8, 8 * FD * 4));
  a.g_pre = off;
  off += a128((Gq * FD + 2048 + SINK_STAGE) * 4);   // next unit's queries, centroids, sink indices
  a.g_bytes = off;
  a.dstride = two_dstride(L, k, S);
  return a;
}

// the forced bitmaps stay in shared memory unless that is what keeps the kernel from fitting
// (moving them to global memory to get C2 under the 164 KB carveout measured 1.5% slower)
static bool two_forced_smem(int64_t L, int k, int S, int cap, int Gq) {
  return TBL_BYTES + 2 * two_layout(L, k, S, cap, Gq, true).g_bytes <= 227 * 1024;
}

int two_select_smem_bytes(int64_t L, int k, int S, int cap, int Gq) {
  return TBL_BYTES + 2 * two_layout(L, k, S, cap, Gq, two_forced_smem(L, k, S, cap, Gq)).g_bytes;
}
static int attend_smem(int nw, int Gq, bool rec16) {
  return std::max(nw * ATT_STAGES * (rec16 ? STAGE16_BYTES : STAGE_BYTES), nw * Gq * (FD + 2) * 4);
}
int two_attend_smem_bytes(int64_t L, int k, int S, int Gq, bool rec16) {   // the wider CTA (the bound)
  (void)L; (void)k; (void)S;
  return attend_smem(ATT_WARPS_MAX, Gq, rec16);
}
static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }
// attention CTAs per unit: enough CTAs for four per SM when the units alone are too few
constexpr int kMaxSplit = 8;
constexpr int64_t kSplitUnits = 1024;   // workspace for split partials up to this many units
static int two_nsplit(int64_t U, int nsm, int nw) {
  // split when the units are fewer than four per SM whatever the CTA width (with 2-warp CTAs
  // a threshold of eight per SM split the 8-GPU C4 shard, 896 units: 0.118 -> 0.147 ms)
  (void)nw;
  const int64_t slots = (int64_t)att_ctas_per_sm(ATT_WARPS_MAX) * nsm;
  if (U >= slots || U > kSplitUnits) return 1;
  return (int)std::min<int64_t>(kMaxSplit, (slots + U - 1) / U);
}
static size_t split_bytes(int64_t U) {
  return U > kSplitUnits ? 0 : a256((size_t)U * kMaxSplit * 8 * (FD + 2) * 4) + a256((size_t)U * 4);
}
size_t two_workspace_bytes(int64_t U, int64_t L, int k, int S) {
  const int64_t W = (L + 31) / 32;
  return 256 + a256((size_t)U * 4) + a256((size_t)U * two_dstride(L, k, S) * 4) + a256((size_t)U * 2 * W * 4) +
         a256((size_t)U * W * 4) + split_bytes(U);
}

cudaError_t launch_decode_two(const uint8_t* signs, const uint8_t* recs, const float* cent32, const float* alpha32,
                              const int32_t* sink_idx, int S, const uint32_t* ffrag, int fblocks,
                              const int32_t* rn, int R,
                              const float* q, int64_t U, int64_t L, int Gq, int k, int cap, float* out, float* lse,
                              int32_t* sel, int sel_stride, int32_t* sel_count, int32_t* diag, void* workspace,
                              int nsm, const int32_t* umap, int mode, const sikv_exchange* xchg, cudaStream_t st) {
  const int lut_mode = mode & 1;
  const bool rec16 = (mode & 2) != 0;
  TwoArgs a = two_layout(L, k, S, cap, Gq, two_forced_smem(L, k, S, cap, Gq));
  a.signs = signs; a.recs = recs; a.cent32 = cent32; a.alpha32 = alpha32; a.sink_idx = sink_idx;
  a.ffrag = ffrag; a.rn = rn; a.umap = umap; a.q = q; a.out = out; a.lse = lse; a.sel = sel; a.sel_count = sel_count; a.diag = diag;
  char* ws = reinterpret_cast<char*>(workspace) + 256;
  a.ndyn = reinterpret_cast<int32_t*>(ws);
  ws += a256((size_t)U * 4);
  a.dynl = reinterpret_cast<int32_t*>(ws);
  ws += a256((size_t)U * a.dstride * 4);
  a.gbits = reinterpret_cast<uint32_t*>(ws);
  ws += a256((size_t)U * 2 * ((L + 31) / 32) * 4);
  a.gforced = reinterpret_cast<uint32_t*>(ws);
  ws += a256((size_t)U * ((L + 31) / 32) * 4);
  const int nw = att_warps(U, L, k, S, nsm);
  a.nsplit = two_nsplit(U, nsm, nw);
  if (a.nsplit > 1) {
    a.spart = reinterpret_cast<float*>(ws);
    a.scnt = reinterpret_cast<int32_t*>(ws + a256((size_t)U * kMaxSplit * 8 * (FD + 2) * 4));
  }
  a.L = L; a.U = U; a.fblocks = fblocks; a.S = S; a.R = R; a.Gq = Gq; a.k = k; a.sel_stride = sel_stride;
  a.lut_mode = lut_mode;
  // the exchange rides on the attention epilogue (measured against a push kernel launched
  // after the attention with PDL: C2 / 8 ranks +8.4 vs +8.8 us, C4 +7.8 vs +7.2 us)
  a.x = xchg ? *xchg : sikv_exchange{};
  const int smem_s = TBL_BYTES + 2 * a.g_bytes;
  auto select = (L + 255) / 256 >= 256 ? decode_select_kernel<true> : decode_select_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(select, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(nsm, (U + 1) / 2);
  select<<<grid, SEL_THREADS, smem_s, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int smem_a = attend_smem(nw, Gq, rec16);
  auto pick = [&](auto w) {
    constexpr int W = decltype(w)::value;
    if (a.x.npeers)
      return a.nsplit > 1 ? (rec16 ? decode_attend_kernel<true, true, W, true> : decode_attend_kernel<false, true, W, true>)
                          : (rec16 ? decode_attend_kernel<true, false, W, true> : decode_attend_kernel<false, false, W, true>);
    return a.nsplit > 1 ? (rec16 ? decode_attend_kernel<true, true, W> : decode_attend_kernel<false, true, W>)
                        : (rec16 ? decode_attend_kernel<true, false, W> : decode_attend_kernel<false, false, W>);
  };
  auto attend = nw == 2 ? pick(std::integral_constant<int, 2>()) : pick(std::integral_constant<int, ATT_WARPS_MAX>());
  e = cudaFuncSetAttribute(attend, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(U * a.nsplit));
  cfg.blockDim = dim3(32 * nw);
  cfg.dynamicSmemBytes = (size_t)smem_a;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attend, a);
}

}  // namespace sikv
