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
//   decode_attend_kernel   one 256-thread CTA per unit, two per SM: the unit's dynamic list,
//                          forced rows and sparse flash-decode (decode_common.cuh), fixed-order
//                          merge, output.
//
// The arithmetic is that of decode.cu (shared device code): selections are identical, the
// outputs equal within float32 accumulation order (the dynamic list is emitted in segment
// order by 8-warp groups exactly as decode.cu does, so they are in fact bit-identical).
#include "common.cuh"
#include "select.cuh"
#include "api_types.cuh"
#include "decode_common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>

namespace sikv {

constexpr int SEL_THREADS = 512;
#ifndef SIKV_PDL
#define SIKV_PDL 1   // attention launched as a programmatic dependent of the selection grid
#endif
__device__ long long* g_prof_two = nullptr;   // optional per-unit phase clocks (profiling)
#ifndef SIKV_SEL_SKS
#define SIKV_SEL_SKS 0
#endif
constexpr bool SEL_SKS = SIKV_SEL_SKS;
// the selection groups' radix digit: 9 bits (512 bins) — at C4 (1.4 K candidates per unit)
// 2.5% faster than 11 bits, neutral at C2; path 1 keeps 11 bits (C3: 6 K candidates)
#ifndef SIKV_SEL_RB
#define SIKV_SEL_RB 9
#endif
constexpr int SEL_NBIN = 1 << SIKV_SEL_RB;    // sample keys in shared memory (A/B: slower at C2)
using SG0 = NamedGroup<1, 0>;
using SG1 = NamedGroup<2, 256>;

struct TwoArgs {
  CUtensorMap recs_map;   // records as a [U*L][128 B] 2-D tensor: TMA gather4 of attention rows
  const uint8_t* signs;
  const uint8_t* recs;
  const float* cent32;
  const float* alpha32;
  const int32_t* sink_idx;
  const uint32_t* ffrag;
  const int32_t* rn;    // [U] recent rows per unit, nullable (then R)
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
  int64_t L, U;
  int fblocks, S, R, Gq, k, capw, sel_stride, dstride;
  int lut_mode;         // 0: centroid LUT, 1: sign-only LUT
  // select-kernel shared-memory layout (per group: misc | hist | forced | cand)
  int g_bytes, g_hist, g_forced, g_cand, g_sks, g_pre;   // g_forced < 0: forced bitmap in gforced
};

// ---------------------------------------------------------------- selection
// the group's staging area for the next unit's queries and centroids (cp.async)
__device__ __forceinline__ void prefetch_unit(const TwoArgs& a, char* base, int tid, int64_t un) {
  const uint32_t pre_s = (uint32_t)__cvta_generic_to_shared(base + a.g_pre);
  if (un >= 0 && un < a.U) {
    for (int i = tid; i < a.Gq * FD / 4; i += DT)
      cp_async16_s(pre_s + 16u * (uint32_t)i, a.q + un * a.Gq * FD + 4 * i);
    for (int i = tid; i < 512; i += DT)
      cp_async16_s(pre_s + (uint32_t)(a.Gq * FD * 4) + 16u * (uint32_t)i, a.cent32 + un * 2048 + 4 * i);
  }
  cp_commit();
}

// one unit's selection by one 8-warp group: the unit's queries / centroids were prefetched
// into the staging area; `next` (or -1) is prefetched once they have been consumed.
// Returns the dynamic list length (the list is in a.dynl).
template <class PG, int G>
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
  uint32_t* sks = reinterpret_cast<uint32_t*>(base + a.g_sks);
  const float* pre_q = reinterpret_cast<const float*>(base + a.g_pre);   // [8][128]
  const float4* pre_c = reinterpret_cast<const float4*>(pre_q + Gq * FD);  // [512]
  long long* prof = g_prof_two ? g_prof_two + u * 12 : nullptr;
  if (prof && tid == 0) prof[0] = clock64();
  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + u * L * FSIGN);
  const UnitGeom g = unit_geom(L, S, a.k, a.capw, a.sink_idx + u * S);
  const int psid = tid < S ? a.sink_idx[u * S + tid] : -1;
  uint4 wsamp[MAX_SAMPLE_CHUNKS];
  load_sample(g, signs, tid, wsamp);
  uint32_t* forced = a.g_forced >= 0 ? forced_s : a.gforced + u * W;
  const float* qs = pre_q;
  cp_wait<0>();                      // this unit's queries / centroids have landed
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  PG::sync();
  if (psid >= 0) atomicOr(&forced[psid >> 5], 1u << (psid & 31));
  for (int j = tid + DT; j < S; j += DT) {
    const int t = a.sink_idx[u * S + j];
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
    fb = produce_candidates<PG, NoX, ColKey, NB, SEL_SKS>(g, signs, T, forced, wsamp, cand, th, tmin, ms, tau, NoX(),
                                                           sks) ? 1 : 0;
    if (prof && tid == 0) prof[2] = clock64();
    if (!fb) {
      ndyn = select_emit_candidates<PG, SEL_NBIN>(g, forced, cand, ms->wcnt, ms->maxx, tau, hist, ms, gt, eq, dyn, sel_u,
                                        a.rn ? __ldg(a.rn + u) : a.R, sel_count_u, kstar);
    } else {
      produce_exact<PG, NoX, ColKey, SEL_NBIN>(g, signs, T, forced, hist, ms, gt, eq, kstar, need_eq, eq_count);
    }
  }
  if (ndyn < 0)
    ndyn = emit_selection<PG>(g, mode, forced, gt, eq, need_eq, eq_count, dyn, sel_u, a.rn ? __ldg(a.rn + u) : a.R,
                              sel_count_u, ms);
  if (prof && tid == 0) prof[3] = clock64();
  if (tid == 0) {
    a.ndyn[u] = ndyn;
    if (a.diag) a.diag[u] = (mode & 3) | (fb ? 4 : 0);
  }
  PG::sync();                       // the group's shared memory is reused by its next unit
  return ndyn;
}

template <class PG, int G>
__device__ __forceinline__ void select_group(const TwoArgs& a, char* sm) {
  prefetch_unit(a, sm + TBL_BYTES + G * a.g_bytes, PG::tid(), (int64_t)blockIdx.x + (int64_t)G * gridDim.x);
  for (int it = 0;; ++it) {
    const int64_t u = (int64_t)blockIdx.x + (int64_t)(2 * it + G) * gridDim.x;
    if (u >= a.U) break;
    select_unit<PG, G>(a, sm, u, u + 2 * gridDim.x);
  }
}

__global__ void __launch_bounds__(SEL_THREADS, 1) decode_select_kernel(TwoArgs a) {
  extern __shared__ __align__(128) char sm[];
#if SIKV_PDL
  // the attention grid may be scheduled onto SMs as this grid's CTAs retire: it attends the
  // forced rows, then waits for this grid to complete (griddepcontrol.wait) before the lists
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  // group from a value the compiler can prove warp-uniform (uniform-datapath table base)
  const int grp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 8), 0);
  if (grp == 0) select_group<SG0, 0>(a, sm);
  else select_group<SG1, 1>(a, sm);
}

// ---------------------------------------------------------------- attention
#ifndef SIKV_ATT_WARPS
#define SIKV_ATT_WARPS 4
#endif
constexpr int ATT_WARPS = SIKV_ATT_WARPS;          // warps per attention CTA (one unit each)
constexpr int ATT_THREADS = 32 * ATT_WARPS;
constexpr int ATT_CTAS_PER_SM = 16 / ATT_WARPS;
#ifndef SIKV_TMA_GATHER
#define SIKV_TMA_GATHER 0   // 1: attention rows staged by TMA tile::gather4 (measured 5% slower than cp.async)
#endif
#ifndef SIKV_ATT_STAGES
#define SIKV_ATT_STAGES 2     // cp.async staging buffers per warp
#endif
constexpr int ATT_STAGES = SIKV_ATT_STAGES;
#ifndef SIKV_TMA_STAGES
#define SIKV_TMA_STAGES 2
#endif
constexpr int TMA_STAGES = SIKV_TMA_STAGES;
#ifndef SIKV_ATT_PREFETCH
#define SIKV_ATT_PREFETCH 1
#endif

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT;\n}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
// four 128-B rows (tensor rows r0..r3) into 512 contiguous bytes at dst, 128-B swizzled
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int r0, int r1, int r2,
                                            int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// Dynamic rows staged by TMA: per 16-token block, lanes 0-3 each issue one gather4 (four
// indexed rows, 512 B) onto the block's mbarrier; two 2 KiB buffers per warp (1 KiB aligned).
// The hardware 128-B swizzle puts chunk k of smem row s at slot k ^ (s & 7); token j of the
// block sits in smem row P(j) = j ^ ((j & 1) << 2) (an involution), so that the fragment reads
// of attn_block stay conflict-free: tokens 2q / 2q + 1 differ in bit 2 of their row (K reads),
// and tokens 0, 2, 4, 6 (and 1, 3, 5, 7) differ in bits 1-2 (V reads).
__device__ __forceinline__ int tma_row(int j) { return j ^ ((j & 1) << 2); }

__device__ __forceinline__ void attn_dynamic_tma(Attn& A, const CUtensorMap* map, int row0, const int32_t* dyn,
                                                 int ndyn, int first, int nw, char* stage, uint32_t bars,
                                                 int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  const int nbd = (ndyn + 15) >> 4;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage);
  const int jv0 = 2 * t4, jv1 = 2 * t4 + 1;
  const int rk = tma_row(g), r0 = tma_row(jv0), r1 = tma_row(jv1);
  BlkOffs o;
  o.k4 = rk * FREC + 16 * (t4 ^ rk);
  o.kp = rk * FREC + 16 * (6 ^ rk);
  o.vw0 = r0 * FREC + 16 * ((4 + (g >> 2)) ^ r0) + 4 * (g & 3);
  o.vw1 = r1 * FREC + 16 * ((4 + (g >> 2)) ^ r1) + 4 * (g & 3);
  o.vp0 = r0 * FREC + 16 * (7 ^ r0);
  o.vp1 = r1 * FREC + 16 * (7 ^ r1);
  // lane l < 4 stages smem rows 4l .. 4l + 3: tokens tma_row(4l + i) (rows >= 8: + 8)
  int ix[4];
  auto load_ix = [&](int blk) {
    if (lane < 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int srow = 4 * lane + i;
        ix[i] = dyn[blk * 16 + (tma_row(srow & 7) | (srow & 8))];
      }
    }
  };
  auto stage_blk = [&](int buf) {
    if (lane < 4) {
      const uint32_t bar = bars + 8u * (uint32_t)buf;
      if (lane == 0) mbar_expect_tx(bar, 16 * FREC);
      tma_gather4(sbase + (uint32_t)(buf * STAGE_BYTES + 512 * lane), map, bar, row0 + ix[0], row0 + ix[1],
                  row0 + ix[2], row0 + ix[3]);
    }
  };
  uint32_t phase = 0;   // bit b: parity of buffer b's next completion
#pragma unroll
  for (int s = 0; s < TMA_STAGES - 1; ++s) {
    if (first + s * nw < nbd) { load_ix(first + s * nw); stage_blk(s); }
  }
  if (first + (TMA_STAGES - 1) * nw < nbd) load_ix(first + (TMA_STAGES - 1) * nw);
  int buf = 0;
  for (int db = first; db < nbd; db += nw) {
    const int nx = db + (TMA_STAGES - 1) * nw;
    if (nx < nbd) {
      stage_blk(buf == 0 ? TMA_STAGES - 1 : buf - 1);
      if (nx + nw < nbd) load_ix(nx + nw);
    }
    mbar_wait(bars + 8u * (uint32_t)buf, (phase >> buf) & 1u);
    phase ^= 1u << buf;
    attn_block(A, stage + buf * STAGE_BYTES, o, ndyn - db * 16, lane);
    __syncwarp();
    buf = buf + 1 == TMA_STAGES ? 0 : buf + 1;
  }
}

// One unit's attention by one CTA of NW warps.  Every warp starts on its own: q~ and the row
// indices come straight from global memory (L2), so the only CTA-wide barriers are the
// two around the partial merge.
template <int NW>
__device__ __forceinline__ void attend_unit(const TwoArgs& a, char* stage, int64_t u) {
  constexpr int NT = 32 * NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if SIKV_TMA_GATHER
  // 1 KiB-aligned staging (128-B swizzle atoms), then the 2 mbarriers per warp
  {
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(stage);
    stage += (1024u - (s0 & 1023u)) & 1023u;
  }
  const int core = max(NW * TMA_STAGES * STAGE_BYTES, NW * a.Gq * (FD + 2) * 4);   // staging, then merge partials
  const uint32_t bars = (uint32_t)__cvta_generic_to_shared(stage + ((core + 7) & ~7));
  if (tid < TMA_STAGES * NW) mbar_init(bars + 8u * (uint32_t)tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
#endif
  const int S = a.S, R = a.rn ? __ldg(a.rn + u) : a.R, Gq = a.Gq;
  const int32_t* dyn = a.dynl + u * a.dstride;
  const int nf = S + R;
  const int nbf = (nf + 15) >> 4;
  const uint32_t* ffrag_u = a.ffrag + u * a.fblocks * FBLK_WORDS;
#if SIKV_ATT_PREFETCH
  // start the forced fragments and the list on their way to L2 while q~ loads
  for (int i = tid; i < (nbf * FBLK_WORDS * 4 + 127) / 128; i += NT)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(ffrag_u) + 128 * i));
  for (int i = tid; i < a.dstride / 32; i += NT)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(dyn) + 128 * i));
#endif
  Attn A;
  attn_init_g(A, a.q + u * Gq * FD, a.alpha32 + u * FD, Gq, lane);
  attn_forced(A, ffrag_u, nf, warp, NW, lane);
#if SIKV_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the selection grid is complete
#endif
  const int ndyn = __ldg(a.ndyn + u);
#if SIKV_TMA_GATHER
  attn_dynamic_tma(A, &a.recs_map, (int)(u * a.L), dyn, ndyn, (warp - nbf % NW + NW) % NW, NW,
                   stage + warp * TMA_STAGES * STAGE_BYTES, bars + 8u * TMA_STAGES * (uint32_t)warp, lane);
#else
  attn_dynamic<ATT_STAGES>(A, a.recs + u * a.L * FREC, dyn, ndyn, (warp - nbf % NW + NW) % NW, NW,
                           stage + warp * ATT_STAGES * STAGE_BYTES, lane);
#endif
  __syncthreads();
  float* part = reinterpret_cast<float*>(stage);
  float* pm = part + NW * Gq * FD;
  float* pl = pm + NW * Gq;
  attn_write_partial(A, part, pm, pl, warp, Gq, lane);
  __syncthreads();
  attn_merge<Cta256>(part, pm, pl, NW, Gq, tid, NT, a.out + u * Gq * FD, a.lse ? a.lse + u * Gq : nullptr);
}

__global__ void __launch_bounds__(ATT_THREADS, ATT_CTAS_PER_SM) decode_attend_kernel(const __grid_constant__ TwoArgs a) {
  extern __shared__ __align__(128) char sm[];
  attend_unit<ATT_WARPS>(a, sm, blockIdx.x);
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
  a.g_sks = off;
  off += SEL_SKS ? MAX_SAMPLE_CHUNKS * DT * 4 : 0;
  a.g_pre = off;
  off += a128((Gq * FD + 2048) * 4);      // next unit's queries and centroids
  a.g_bytes = off;
  a.dstride = two_dstride(L, k, S);
  return a;
}

// the forced bitmaps stay in shared memory unless that is what keeps the kernel from fitting
// (moving them to global memory to get C2 under the 164 KB carveout measured 1.5% slower)
static bool two_forced_smem(int64_t L, int k, int S, int cap, int Gq) {
  return TBL_BYTES + 2 * two_layout(L, k, S, cap, Gq, true).g_bytes <= 227 * 1024;
}

#ifndef SIKV_SEL_PAD
#define SIKV_SEL_PAD 0
#endif
int two_select_smem_bytes(int64_t L, int k, int S, int cap, int Gq) {
  return TBL_BYTES + 2 * two_layout(L, k, S, cap, Gq, two_forced_smem(L, k, S, cap, Gq)).g_bytes + SIKV_SEL_PAD;
}
int two_attend_smem_bytes(int64_t L, int k, int S, int Gq) {
  const int st = SIKV_TMA_GATHER ? TMA_STAGES : ATT_STAGES;
  const int core = std::max(ATT_WARPS * st * STAGE_BYTES, ATT_WARPS * Gq * (FD + 2) * 4);
  return SIKV_TMA_GATHER ? ((core + 7) & ~7) + 8 * TMA_STAGES * ATT_WARPS + 1024 : core;   // mbarriers, 1 KiB alignment slack
}
static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }
size_t two_workspace_bytes(int64_t U, int64_t L, int k, int S) {
  const int64_t W = (L + 31) / 32;
  return 256 + a256((size_t)U * 4) + a256((size_t)U * two_dstride(L, k, S) * 4) + a256((size_t)U * 2 * W * 4) +
         (size_t)U * W * 4;
}

cudaError_t launch_decode_two(const uint8_t* signs, const uint8_t* recs, const float* cent32, const float* alpha32,
                              const int32_t* sink_idx, int S, const uint32_t* ffrag, int fblocks,
                              const int32_t* rn, int R,
                              const float* q, int64_t U, int64_t L, int Gq, int k, int cap, float* out, float* lse,
                              int32_t* sel, int sel_stride, int32_t* sel_count, int32_t* diag, void* workspace,
                              int nsm, int lut_mode, cudaStream_t st) {
  TwoArgs a = two_layout(L, k, S, cap, Gq, two_forced_smem(L, k, S, cap, Gq));
  a.signs = signs; a.recs = recs; a.cent32 = cent32; a.alpha32 = alpha32; a.sink_idx = sink_idx;
  a.ffrag = ffrag; a.rn = rn; a.q = q; a.out = out; a.lse = lse; a.sel = sel; a.sel_count = sel_count; a.diag = diag;
  char* ws = reinterpret_cast<char*>(workspace) + 256;
  a.ndyn = reinterpret_cast<int32_t*>(ws);
  ws += a256((size_t)U * 4);
  a.dynl = reinterpret_cast<int32_t*>(ws);
  ws += a256((size_t)U * a.dstride * 4);
  a.gbits = reinterpret_cast<uint32_t*>(ws);
  ws += a256((size_t)U * 2 * ((L + 31) / 32) * 4);
  a.gforced = reinterpret_cast<uint32_t*>(ws);
#if SIKV_TMA_GATHER
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)FREC, (cuuint64_t)(U * L)};
    const cuuint64_t strides[1] = {(cuuint64_t)FREC};
    const cuuint32_t box[2] = {(cuuint32_t)FREC, 1};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&a.recs_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(recs), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
#endif
  a.L = L; a.U = U; a.fblocks = fblocks; a.S = S; a.R = R; a.Gq = Gq; a.k = k; a.sel_stride = sel_stride;
  a.lut_mode = lut_mode;
  const int smem_s = TBL_BYTES + 2 * a.g_bytes + SIKV_SEL_PAD;
  cudaError_t e = cudaFuncSetAttribute(decode_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(nsm, (U + 1) / 2);
  decode_select_kernel<<<grid, SEL_THREADS, smem_s, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int smem_a = two_attend_smem_bytes(L, k, S, Gq);
  e = cudaFuncSetAttribute(decode_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a);
  if (e != cudaSuccess) return e;
#if SIKV_PDL
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)U);
  cfg.blockDim = dim3(ATT_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem_a;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_attend_kernel, a);
#else
  decode_attend_kernel<<<(unsigned)U, ATT_THREADS, smem_a, st>>>(a);
  return cudaGetLastError();
#endif
}

}  // namespace sikv
