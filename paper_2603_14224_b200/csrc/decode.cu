// Fused decode step for the self-indexing KV cache (sm_100a): one CTA per decode unit
// (layer x batch x KV head).
//
//   A  q-bar = sum of the GQA group's queries; LUT[g][c] = q-bar_g . centroid[g][c]
//      (retrieval.py:46-51) and the byte-pair table T[b][p] = LUT[2p][b&15] + LUT[2p+1][b>>4]
//   B  score every prefill token from its 16-byte sign record (retrieval.py:65-77):
//      16 pair lookups, conflict-free (each half warp's 16 lanes hit 16 distinct banks
//      because lane j starts at pair j and the plane is stored pre-rotated by t mod 16)
//   C  exact top-k of the non-forced tokens, ties -> lower index (retrieval.py:127-161):
//      a sampled threshold keeps only ~1.5k candidates in shared memory, then a radix
//      select finds the k-th key; an exact multi-pass radix path covers the rare case
//      where the sampled threshold over- or under-shoots
//   D  sparse flash-decode over sinks + recents + the k selected tokens
//      (attention.py:35-62): K / V dequantised straight into mma.sync m16n8k16 fragments
//      (alpha folded into the query, sign applied by one LOP3 per pair), online softmax,
//      fixed-order merge of the 8 warp partials.
#include "common.cuh"
#include "select.cuh"
#include "decode_common.cuh"
#include "api_types.cuh"
#include <math.h>
#include <algorithm>

namespace sikv {

constexpr int K1_STAGES = 2;             // cp.async stages per warp in the attention phase
__device__ long long* g_prof = nullptr;
__device__ int g_k1_skip = 0;            // debug: bit 0 skips the attention phase   // optional per-unit phase clocks (debug / profiling)

struct DecodeArgs {
  const uint8_t* signs;     // [U][L][16] rotated sign plane
  const uint8_t* recs;      // [U][L][128] records
  const float* cent32;      // [U][32][16][4]
  const float* alpha32;     // [U][128]
  const int32_t* sink_idx;  // [U][S] sorted, unique, < L
  const uint32_t* ffrag;    // [U][fblocks][FBLK_WORDS] forced rows: fp16 fragments + row scales
  const int32_t* rn;        // [U] recent rows per unit, nullable (then R for every unit)
  const int32_t* umap;      // [U] cache unit of each query unit (per-q-head policy), nullable = identity
  const float* q;           // [U][Gq][128]
  float* out;               // [U][Gq][128]
  float* lse;               // [U][Gq] natural-log sum of exp(logits), nullable
  int32_t* sel;             // [U][sel_stride], nullable
  int32_t* sel_count;       // [U], nullable
  int32_t* diag;            // [U], nullable
  int64_t L;
  int fblocks;
  int S, R, Gq, k, capw, sel_stride;
  int lut_mode;             // 0: centroid LUT, 1: sign-only LUT
  // shared-memory layout (byte offsets)
  int off_cand, off_forced, off_misc, off_bits, off_dyn, off_stage;
};

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(DT, 2) decode_step_kernel(DecodeArgs a) {
  extern __shared__ __align__(128) char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t u = blockIdx.x;
  const int64_t L = a.L;
  char* T = sm;                                                   // R0: pair table
  uint32_t* cand = reinterpret_cast<uint32_t*>(sm + a.off_cand);  // R1: per-warp (x, t) segments
  uint32_t* forced = reinterpret_cast<uint32_t*>(sm + a.off_forced);
  Misc* ms = reinterpret_cast<Misc*>(sm + a.off_misc);
  float* qs = reinterpret_cast<float*>(sm + a.off_misc + 256);    // [Gq][128]
  float* lut = qs + 8 * FD;                                       // [32][16]
  float* qbar = lut + 512;                                        // [128]
  float* inva = qbar + FD;                                        // [128] 1 / alpha-hat
  float* ahat = inva + FD;                                        // [128] alpha-hat
  const int64_t cu = a.umap ? (int64_t)a.umap[u] : u;              // the unit's cache
  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + cu * L * FSIGN);
  const int S = a.S, R = a.rn ? a.rn[cu] : a.R, Gq = a.Gq;
  const int W = (int)((L + 31) >> 5);
  long long* prof = g_prof ? g_prof + u * 16 : nullptr;
#define PROF(i) do { if (prof && tid == 0) prof[i] = clock64(); } while (0)
  PROF(0);
  const UnitGeom g = unit_geom(L, S, a.k, a.capw, a.sink_idx + cu * S);
  // every small per-unit input is in flight at once, before any shared-memory step
  float pq[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pq[i] = tid + DT * i < Gq * FD ? a.q[u * Gq * FD + tid + DT * i] : 0.f;
  const float pal = tid < FD ? a.alpha32[cu * FD + tid] : 0.f;
  const float4* c4 = reinterpret_cast<const float4*>(a.cent32 + cu * 32 * 16 * 4);
  const float4 pc0 = c4[tid], pc1 = c4[tid + DT];
  const int psid = tid < S ? a.sink_idx[cu * S + tid] : -1;
  uint4 wsamp[MAX_SAMPLE_CHUNKS];      // the sample's loads overlap the setup below
  load_sample(g, signs, tid, wsamp);

  // ---------------- A: queries, LUT, pair table, forced bitmap
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (tid + DT * i < Gq * FD) qs[tid + DT * i] = pq[i];
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  if (tid == 0) ms->fb = 0;
  __syncthreads();
  if (psid >= 0) atomicOr(&forced[psid >> 5], 1u << (psid & 31));
  for (int j = tid + DT; j < S; j += DT) {
    const int t = a.sink_idx[cu * S + j];
    atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  if (tid < FD) {
    float s = qs[tid];
    for (int h = 1; h < Gq; ++h) s = __fadd_rn(s, qs[h * FD + tid]);
    qbar[tid] = s;
    ahat[tid] = pal > 0.f ? pal : 1.0f;
    inva[tid] = 1.0f / ahat[tid];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = tid + DT * r, gg = e >> 4;
    const float4 c = lut_factors(r ? pc1 : pc0, e & 15, a.lut_mode);
    const float q0 = qbar[4 * gg], q1 = qbar[4 * gg + 1], q2 = qbar[4 * gg + 2], q3 = qbar[4 * gg + 3];
    lut[(e & 15) * 32 + gg] = __fadd_rn(__fadd_rn(__fmul_rn(q0, c.x), __fmul_rn(q2, c.z)),
                                        __fadd_rn(__fmul_rn(q1, c.y), __fmul_rn(q3, c.w)));
  }
  __syncthreads();
  build_pair_rows<Cta256>(lut, T);
  PROF(1);

  // ---------------- B/C: candidates, exact k-th key, tie-aware bitmaps
  const int mode = g.mode;
  uint32_t* gt = reinterpret_cast<uint32_t*>(sm + a.off_bits);   // R0 once the table is dead
  uint32_t* eq = gt + W;
  uint32_t kstar = 0;
  int need_eq = 0, eq_count = 0;
  int ndyn = -1;
  int32_t* sel_u = a.sel ? a.sel + u * a.sel_stride : nullptr;
  int32_t* sel_count_u = a.sel_count ? a.sel_count + u : nullptr;
  if (mode >= 2) {
    uint32_t tau;
    const bool fb = produce_candidates<Cta256>(g, signs, T, forced, wsamp, cand, reinterpret_cast<int*>(cand),
                                               cand + 256, ms, tau);
    PROF(3);
    if (!fb) {
      ndyn = select_emit_candidates<Cta256>(g, forced, cand, ms->wcnt, ms->maxx, tau, reinterpret_cast<int*>(T), ms,
                                            gt, eq, reinterpret_cast<int32_t*>(sm + a.off_dyn), sel_u, R,
                                            sel_count_u, kstar);
    } else {
      if (tid == 0) ms->fb = 1;
      gt = cand + NBIN + 64;                                      // R1: candidates are void
      eq = gt + W;
      produce_exact<Cta256>(g, signs, T, forced, reinterpret_cast<int*>(cand), ms, gt, eq, kstar, need_eq,
                            eq_count);
    }
  }
  PROF(4);
  if (ndyn < 0)
    ndyn = emit_selection<Cta256>(g, mode, forced, gt, eq, need_eq, eq_count,
                                  reinterpret_cast<int32_t*>(sm + a.off_dyn), sel_u, R, sel_count_u, ms);
  if (tid == 0 && a.diag) a.diag[u] = (mode & 3) | (ms->fb ? 4 : 0);

  PROF(5);
  // ---------------- D: sparse attention over forced rows + dynamic rows
  Attn A;
  attn_init(A, qs, ahat, Gq, lane);
  const int nf = S + R;
  const int nbf = (nf + 15) >> 4;
  if (g_k1_skip & 1) return;
  attn_forced(A, a.ffrag + cu * a.fblocks * FBLK_WORDS, nf, warp, DW, lane);
  PROF(6);
  attn_dynamic<K1_STAGES>(A, a.recs + cu * L * FREC, reinterpret_cast<const int32_t*>(sm + a.off_dyn), ndyn,
                          (warp - nbf % DW + DW) % DW, DW, sm + warp * K1_STAGES * STAGE_BYTES, lane);
  PROF(7);
  // ---------------- merge the 8 warp partials (fixed order)
  __syncthreads();
  PROF(8);
  float* part = reinterpret_cast<float*>(cand);           // [DW][Gq][128]
  float* pm = part + DW * Gq * FD;                         // [DW][Gq]
  float* pl = pm + DW * Gq;                                // [DW][Gq]
  attn_write_partial(A, part, pm, pl, warp, Gq, lane);
  __syncthreads();
  attn_merge<Cta256>(part, pm, pl, DW, Gq, tid, DT, a.out + u * Gq * FD, a.lse ? a.lse + u * Gq : nullptr);
  PROF(9);
#undef PROF
}

// ---------------------------------------------------------------- scores only (tests / API)
__global__ void score_fast_kernel(const uint8_t* __restrict__ signs_, const float* __restrict__ cent32,
                                  const float* __restrict__ q, int Gq, int64_t L, int lut_mode,
                                  float* __restrict__ out) {
  extern __shared__ __align__(16) char T[];                  // TBL_BYTES
  __shared__ float lut[512];
  __shared__ float qbar[FD];
  const int64_t u = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < FD) {
    float s = q[u * Gq * FD + tid];
    for (int h = 1; h < Gq; ++h) s = __fadd_rn(s, q[(u * Gq + h) * FD + tid]);
    qbar[tid] = s;
  }
  __syncthreads();
  const float* C = cent32 + u * 2048;
  for (int e = tid; e < 512; e += blockDim.x) {
    const int g = e >> 4;
    const float4 c = lut_factors(reinterpret_cast<const float4*>(C)[e], e & 15, lut_mode);
    lut[e] = __fadd_rn(__fadd_rn(__fmul_rn(qbar[4 * g], c.x), __fmul_rn(qbar[4 * g + 2], c.z)),
                       __fadd_rn(__fmul_rn(qbar[4 * g + 1], c.y), __fmul_rn(qbar[4 * g + 3], c.w)));
  }
  __syncthreads();
  for (int e = tid; e < 4096; e += blockDim.x) {
    const int b = e >> 4, p = e & 15;
    const float v = __fadd_rn(lut[(2 * p) * 16 + (b & 15)], lut[(2 * p + 1) * 16 + (b >> 4)]);
    float* row = reinterpret_cast<float*>(T) + b * 64;
    row[p] = v; row[p + 16] = v; row[p + 32] = v; row[p + 48] = v;
  }
  __syncthreads();
  const uint4* signs = reinterpret_cast<const uint4*>(signs_ + u * L * FSIGN);
  const RepKey lb(lane);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + tid; t < L; t += (int64_t)gridDim.x * blockDim.x)
    out[u * L + t] = score_token(__ldg(signs + t), lb, T);
}

// ---------------------------------------------------------------- host side
static int align128(int x) { return (x + 127) & ~127; }

DecodeLayout decode_layout(int64_t L, int k, int S, int Gq, int cap) {
  DecodeLayout d{};
  const int W = (int)((L + 31) / 32);
  const int keff = (int)std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  d.capw = std::max(32, cap / DW);
  // R0: pair table while scoring; then hist | gt | eq (selection) ... dynamic list at the
  // end; during attention the staging buffers (K1_STAGES per warp) overlay hist / gt / eq
  d.off_bits = align128(NBIN * 4);
  const int stage_end = DW * K1_STAGES * STAGE_BYTES;
  d.off_dyn = align128(std::max(d.off_bits + 2 * W * 4, stage_end));
  d.off_stage = 0;
  const int r0 = std::max(TBL_BYTES, align128(d.off_dyn + (std::max(keff, 1) + 16) * 4));
  // R1: per-warp candidate segments; at other times the tau histogram, the fallback
  // histogram + bitmaps, and the attention partials
  int r1 = DW * d.capw * 8;
  r1 = std::max(r1, (NBIN + 64) * 4 + 2 * W * 4);
  r1 = std::max(r1, DW * Gq * (FD + 2) * 4);
  d.off_cand = align128(r0);
  int off = d.off_cand + align128(r1);
  d.off_forced = off;
  off += align128(W * 4);
  d.off_misc = off;
  off += 256 + (8 * FD + 512 + FD * 3) * 4;
  d.total = align128(off);
  return d;
}

cudaError_t launch_decode(const uint8_t* signs, const uint8_t* recs, const float* cent32,
                          const float* alpha32, const int32_t* sink_idx, int S, const uint32_t* ffrag,
                          int fblocks, const int32_t* rn, int R, const float* q, int64_t U, int64_t L, int Gq, int k, int cap,
                          float* out, float* lse, int32_t* sel, int sel_stride, int32_t* sel_count,
                          int32_t* diag, const int32_t* umap, int lut_mode, cudaStream_t st, int* smem_out) {
  DecodeLayout d = decode_layout(L, k, S, Gq, cap);
  if (smem_out) *smem_out = d.total;
  DecodeArgs a{signs, recs, cent32, alpha32, sink_idx, ffrag, rn, umap, q, out, lse, sel,
               sel_count, diag, L, fblocks, S, R, Gq, k, d.capw, sel_stride, lut_mode,
               d.off_cand, d.off_forced, d.off_misc, d.off_bits, d.off_dyn, d.off_stage};
  cudaError_t e = cudaFuncSetAttribute(decode_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, d.total);
  if (e != cudaSuccess) return e;
  decode_step_kernel<<<(unsigned)U, DT, d.total, st>>>(a);
  return cudaGetLastError();
}

// Forced rows (sinks then recents) -> fp16 mma fragments, one warp per (unit, 16-row block).
// K^ = K' / (alpha-hat * scale) with alpha folded into the query and a power-of-two row scale
// (1 unless the row's |K' / alpha-hat| exceeds 1: recent rows are not bounded by the prefill
// alpha), V as is; rows >= S + R_u are zero.  status bit 2: non-finite entry, bit 4: a V entry
// outside the fp16 range.
__device__ __forceinline__ void pack_block(int64_t u, int blk, int lane, const float* __restrict__ sink_k,
                                           const float* __restrict__ sink_v, int S, const float* rec_k,
                                           const float* rec_v, int64_t rcap, int Ru, const float* __restrict__ alpha32,
                                           int fblocks, uint32_t* __restrict__ frag, int* status, int part = -1) {
  // part: -1 = the whole block; 0 / 1 = the K rows g / g + 8; 2 / 3 = V m-tiles 0-3 / 4-7 (one
  // warp each when a block is packed by four warps)
  const int g = lane >> 2, t4 = lane & 3;
  const int nf = S + Ru;
  auto row = [&](int f, bool key) -> const float* {
    if (f >= nf) return nullptr;
    if (f < S) return (key ? sink_k : sink_v) + (u * S + f) * FD;
    return (key ? rec_k : rec_v) + (u * rcap + (f - S)) * FD;
  };
  auto inva = [&](int d) {
    const float al = alpha32[u * FD + d];
    return 1.0f / (al > 0.f ? al : 1.0f);
  };
  uint32_t* fb = frag + (u * fblocks + blk) * FBLK_WORDS;
  uint32_t* out = fb + lane * 32;
  const int base = blk * 16;
  int bad = 0;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    if (part >= 0 && part != nt) continue;
    const float* kr = row(base + g + 8 * nt, true);
    float x[32];
    float mx = 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int d = 16 * s + 2 * t4 + 8 * e;
        x[4 * s + 2 * e] = kr ? kr[d] * inva(d) : 0.f;
        x[4 * s + 2 * e + 1] = kr ? kr[d + 1] * inva(d + 1) : 0.f;
        mx = fmaxf(mx, fmaxf(fabsf(x[4 * s + 2 * e]), fabsf(x[4 * s + 2 * e + 1])));
      }
    // the row's four lanes (same g) hold all 128 channels
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    if (!(mx <= 3.0e38f)) { bad |= 4; mx = 1.f; }                 // inf / NaN
    float scale = 1.f;
    if (mx > 1.f) { int ex; frexpf(mx, &ex); scale = ldexpf(1.f, ex); }   // mx / scale <= 1
    const float inv = 1.f / scale;
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        out[nt * 16 + 2 * s + e] = h2u(__floats2half2_rn(x[4 * s + 2 * e] * inv, x[4 * s + 2 * e + 1] * inv));
    if (t4 == 0) reinterpret_cast<float*>(fb + 2 * 32 * 32)[g + 8 * nt] = scale;
  }
  uint32_t* ov = out + 32 * 32;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    if (part >= 0 && part != 2 + (m >> 2)) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int d = 16 * m + g + 8 * (r & 1), pr = r >> 1;
      const float* va = row(base + 2 * t4 + 8 * pr, false);
      const float* vb = row(base + 2 * t4 + 8 * pr + 1, false);
      const float a0 = va ? va[d] : 0.f, a1 = vb ? vb[d] : 0.f;
      if (!(fabsf(a0) <= 3.0e38f) || !(fabsf(a1) <= 3.0e38f)) bad |= 4;
      else if (fabsf(a0) > 65504.f || fabsf(a1) > 65504.f) bad |= 16;
      ov[m * 4 + r] = h2u(__floats2half2_rn(a0, a1));
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0 && status) atomicOr(status, bad);
}

__global__ void pack_forced_kernel(const float* __restrict__ sink_k, const float* __restrict__ sink_v, int S,
                                   const float* __restrict__ rec_k, const float* __restrict__ rec_v, int64_t rcap,
                                   const int32_t* __restrict__ rn, int R, const float* __restrict__ alpha32,
                                   int fblocks, int b0, uint32_t* __restrict__ frag, int* status) {
  const int64_t u = blockIdx.y;
  pack_block(u, b0 + blockIdx.x, threadIdx.x & 31, sink_k, sink_v, S, rec_k, rec_v, rcap, rn ? rn[u] : R, alpha32,
             fblocks, frag, status, (int)(threadIdx.x >> 5));
}

cudaError_t launch_pack_forced(const float* sink_k, const float* sink_v, int S, const float* rec_k,
                               const float* rec_v, int64_t rcap, const int32_t* rn, int R, const float* alpha32,
                               int64_t U, int fblocks, int b0, int b1, uint32_t* frag, int* status, cudaStream_t st) {
  if (b1 <= b0 || U == 0) return cudaSuccess;
  pack_forced_kernel<<<dim3(b1 - b0, (unsigned)U), 128, 0, st>>>(sink_k, sink_v, S, rec_k, rec_v, rcap, rn, R,
                                                               alpha32, fblocks, b0, frag, status);
  return cudaGetLastError();
}

// Decode-time append into the forced-row ring (cache.py:274-287 for every listed unit): one
// warp per appended row: recent row rn[u] <- (k - mu, v) as float32 (centred in float64 with
// the frozen prefill mu), the 16-row fragment block holding it re-packed, rn[u] += 1.
__global__ void append_forced_kernel(const void* __restrict__ k, const void* __restrict__ v, int dt, int64_t n,
                                     const int32_t* __restrict__ ids, const double* __restrict__ mu64,
                                     const float* __restrict__ alpha32, const float* __restrict__ sink_k,
                                     const float* __restrict__ sink_v, int S, float* rec_k, float* rec_v,
                                     int64_t rcap, int32_t* rn, int fblocks, uint32_t* __restrict__ frag,
                                     int* status) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t u = ids ? ids[i] : i;
  const int pos = rn[u];
  if (pos >= rcap) {                                     // capacity is the caller's contract
    if (lane == 0 && status) atomicOr(status, 32);
    return;
  }
  int bad = 0;
  for (int d = lane; d < FD; d += 32) {
    const double kd = load_in(k, dt, i * FD + d), vd = load_in(v, dt, i * FD + d);
    if (!isfinite(kd) || !isfinite(vd)) bad = 4;
    rec_k[(u * rcap + pos) * FD + d] = (float)(kd - mu64[u * FD + d]);
    rec_v[(u * rcap + pos) * FD + d] = (float)vd;
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0 && status) atomicOr(status, bad);
  __syncwarp();                                          // the row is visible to the whole warp
  pack_block(u, (S + pos) >> 4, lane, sink_k, sink_v, S, rec_k, rec_v, rcap, pos + 1, alpha32, fblocks, frag, status);
  if (lane == 0) rn[u] = pos + 1;
}

cudaError_t launch_append_forced(const void* k, const void* v, int dt, int64_t n, const int32_t* ids,
                                 const double* mu64, const float* alpha32, const float* sink_k, const float* sink_v,
                                 int S, float* rec_k, float* rec_v, int64_t rcap, int32_t* rn, int fblocks,
                                 uint32_t* frag, int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n + 3) / 4);
  append_forced_kernel<<<blocks, 128, 0, st>>>(k, v, dt, n, ids, mu64, alpha32, sink_k, sink_v, S, rec_k, rec_v, rcap,
                                                rn, fblocks, frag, status);
  return cudaGetLastError();
}

cudaError_t set_k1_skip(int v) { return cudaMemcpyToSymbol(g_k1_skip, &v, sizeof(v)); }
cudaError_t set_decode_profile(long long* p) {
  return cudaMemcpyToSymbol(g_prof, &p, sizeof(p));
}

cudaError_t launch_score_fast(const uint8_t* signs, const float* cent32, const float* q, int Gq,
                              int64_t U, int64_t L, int lut_mode, float* out, cudaStream_t st) {
  const int bx = (int)std::min<int64_t>(64, (L + 255) / 256);
  cudaError_t e = cudaFuncSetAttribute(score_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TBL_BYTES);
  if (e != cudaSuccess) return e;
  score_fast_kernel<<<dim3(bx, (unsigned)U), 256, TBL_BYTES, st>>>(signs, cent32, q, Gq, L, lut_mode, out);
  return cudaGetLastError();
}

}  // namespace sikv
