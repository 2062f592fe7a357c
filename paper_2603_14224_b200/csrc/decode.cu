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
#include "api_types.cuh"
#include <math.h>
#include <algorithm>

namespace sikv {

constexpr int TBL_BYTES = 256 * 64 * 4;   // pair table: 256 byte values x 64 columns

struct DecodeArgs {
  const uint8_t* signs;     // [U][L][16] rotated sign plane
  const uint8_t* recs;      // [U][L][128] records
  const float* cent32;      // [U][32][16][4]
  const float* alpha32;     // [U][128]
  const int32_t* sink_idx;  // [U][S] sorted, unique, < L
  const float* sink_k;      // [U][S][128] centred K'
  const float* sink_v;      // [U][S][128]
  const float* rec_k;       // [U][rcap][128] centred K'
  const float* rec_v;
  const float* q;           // [U][Gq][128]
  float* out;               // [U][Gq][128]
  float* lse;               // [U][Gq] natural-log sum of exp(logits), nullable
  int32_t* sel;             // [U][sel_stride], nullable
  int32_t* sel_count;       // [U], nullable
  int32_t* diag;            // [U], nullable
  int64_t L, rcap;
  int S, R, Gq, k, cap, sel_stride;
  int nsamp;                // sample entries (multiple of 256)
  // shared-memory layout (byte offsets)
  int off_cand, off_samp, off_forced, off_misc, off_lists;
};

// ---------------------------------------------------------------- scoring
// score of the token whose 16-byte rotated sign record is w; lb = byte offset of this
// lane's first column (64*half + 4*j); T = pair table (row stride 256 B).
__device__ __forceinline__ float score_token(const uint4 w, uint32_t lb, const char* T) {
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint32_t off = prmt(ww[i >> 2], lb, 0x5504u | ((uint32_t)(i & 3) << 4));
    float v = *reinterpret_cast<const float*>(T + off + 4 * i);
    s = (i == 0) ? v : __fadd_rn(s, v);
  }
  return s;
}

__device__ __forceinline__ bool forced_bit(const uint32_t* fb, int64_t t) {
  return (fb[t >> 5] >> (t & 31)) & 1u;
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(DT, 1) decode_step_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t u = blockIdx.x;
  const int64_t L = a.L;
  const int W = (int)((L + 31) >> 5);
  char* T = sm;                                                  // pair table (R0)
  uint32_t* cand = reinterpret_cast<uint32_t*>(sm + a.off_cand); // (key, idx) pairs
  uint32_t* samp = reinterpret_cast<uint32_t*>(sm + a.off_samp);
  uint32_t* forced = reinterpret_cast<uint32_t*>(sm + a.off_forced);
  Misc* ms = reinterpret_cast<Misc*>(sm + a.off_misc);
  float* qs = reinterpret_cast<float*>(sm + a.off_misc + 256);   // [Gq][128]
  float* lut = qs + 8 * FD;                                      // [32][16]
  float* qbar = lut + 512;                                       // [128]
  float* inva = qbar + FD;                                       // [128] 1/alpha-hat
  float* ahat = inva + FD;                                       // [128] alpha-hat
  int* hist = reinterpret_cast<int*>(ahat + FD);                 // [256]

  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + u * L * FSIGN);
  const int S = a.S, R = a.R, Gq = a.Gq;

  // ---------------- A: queries, LUT, pair table, forced bitmap
  for (int i = tid; i < Gq * FD; i += DT) qs[i] = a.q[u * Gq * FD + i];
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  if (tid == 0) { ms->ncand = 0; ms->nsv = 0; ms->fb = 0; }
  __syncthreads();
  for (int j = tid; j < S; j += DT) {
    int t = a.sink_idx[u * S + j];
    atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  if (tid < FD) {
    float s = qs[tid];
    for (int h = 1; h < Gq; ++h) s = __fadd_rn(s, qs[h * FD + tid]);
    qbar[tid] = s;
    float al = a.alpha32[u * FD + tid];
    ahat[tid] = al > 0.f ? al : 1.0f;
    inva[tid] = 1.0f / ahat[tid];
  }
  __syncthreads();
  {
    const float* C = a.cent32 + u * 32 * 16 * 4;
    for (int e = tid; e < 512; e += DT) {
      const int g = e >> 4;
      const float4 c = reinterpret_cast<const float4*>(C)[e];
      const float q0 = qbar[4 * g], q1 = qbar[4 * g + 1], q2 = qbar[4 * g + 2], q3 = qbar[4 * g + 3];
      lut[e] = __fadd_rn(__fadd_rn(__fmul_rn(q0, c.x), __fmul_rn(q2, c.z)),
                         __fadd_rn(__fmul_rn(q1, c.y), __fmul_rn(q3, c.w)));
    }
  }
  __syncthreads();
  for (int e = tid; e < 256 * 16; e += DT) {
    const int b = e >> 4, p = e & 15;
    const float v = __fadd_rn(lut[(2 * p) * 16 + (b & 15)], lut[(2 * p + 1) * 16 + (b >> 4)]);
    float* row = reinterpret_cast<float*>(T) + b * 64;
    row[p] = v; row[p + 16] = v; row[p + 32] = v; row[p + 48] = v;
  }
  __syncthreads();

  // candidate bookkeeping
  const int64_t ncand_all = L - S;
  const int keff = (int)((int64_t)a.k < ncand_all ? (int64_t)a.k : ncand_all);
  const uint32_t lb = (uint32_t)(64 * ((lane >> 4) & 1) + 4 * (lane & 15));
  const int nchunks = (int)((L + 255) >> 8);

  // how the selection is found
  //   mode 0: nothing dynamic; mode 1: every candidate selected; mode 2: all candidates fit
  //   (tau = 1); mode 3: sampled threshold
  int mode;
  if (keff == 0) mode = 0;
  else if (keff == ncand_all) mode = 1;
  else if (ncand_all <= a.cap) mode = 2;
  else mode = 3;

  uint32_t* gt = nullptr;
  uint32_t* eq = nullptr;
  uint32_t kstar = 0;
  int need_eq = 0;   // how many key == K* tokens (lowest index first) to take

  auto push_cands = [&](bool pred, uint32_t key, uint32_t t) {
    unsigned m = __ballot_sync(0xffffffffu, pred);
    if (m == 0) return;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(&ms->ncand, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (pred) {
      int pos = base + __popc(m & ((1u << lane) - 1));
      if (pos < a.cap) { cand[2 * pos] = key; cand[2 * pos + 1] = t; }
    }
  };

  bool fallback = false;
  if (mode >= 2) {
    uint32_t tau = 1;
    if (mode == 3) {
      // ---------------- B1: score the sample chunks (every 16th chunk of 256 tokens)
      const int nsc = (nchunks + 15) >> 4;
      for (int c0 = 0; c0 < nsc; c0 += 4) {
        uint4 w[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int64_t t = (int64_t)(c0 + x) * 16 * 256 + tid;
          w[x] = (c0 + x < nsc && t < L) ? __ldg(signs + t) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          if (c0 + x >= nsc) break;
          const int64_t t = (int64_t)(c0 + x) * 16 * 256 + tid;
          uint32_t key = 0;
          if (t < L && !forced_bit(forced, t)) key = f32_key(score_token(w[x], lb, T));
          samp[(c0 + x) * 256 + tid] = key;
          unsigned m = __ballot_sync(0xffffffffu, key != 0);
          if (lane == 0 && m) atomicAdd(&ms->nsv, __popc(m));
        }
      }
      __syncthreads();
      const int nsv = ms->nsv, ns = nsc * 256;
      const double e = (double)keff * (double)nsv / (double)ncand_all;
      int r = (int)ceil(e + 4.0 * sqrt(e) + 16.0);
      r = min(r, nsv);
      if (r >= 1) {
        // radix-select the r-th largest sample key -> tau
        if (tid == 0) ms->rem_sel = r;
        uint32_t prefix = 0, pmask = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
          hist[tid] = 0;
          __syncthreads();
          for (int i0 = 0; i0 < ns; i0 += DT) {
            const int i = i0 + tid;
            const uint32_t key = i < ns ? samp[i] : 0u;
            hist_add(hist, (i < ns && (key & pmask) == prefix) ? (int)((key >> shift) & 255) : -1);
          }
          __syncthreads();
          pick_digit(hist, ms);
          __syncthreads();
          prefix |= (uint32_t)ms->digit << shift;
          pmask |= 0xFFu << shift;
          if (tid == 0) ms->rem_sel -= ms->cnt_above;
          __syncthreads();
        }
        tau = prefix;
      }
      // sample entries at or above tau become candidates
      for (int i0 = 0; i0 < ns; i0 += DT) {
        const int i = i0 + tid;
        const uint32_t key = samp[i];
        const int64_t t = (int64_t)(i >> 8) * 16 * 256 + (i & 255);
        push_cands(key != 0 && key >= tau, key, (uint32_t)t);
      }
      __syncthreads();
    }
    // ---------------- B2: score everything else, keep key >= tau
    for (int c0 = 0; c0 < nchunks; c0 += 4) {
      uint4 w[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int c = c0 + x;
        const int64_t t = (int64_t)c * 256 + tid;
        const bool skip = c >= nchunks || (mode == 3 && (c & 15) == 0);
        w[x] = (!skip && t < L) ? __ldg(signs + t) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int c = c0 + x;
        if (c >= nchunks) break;
        if (mode == 3 && (c & 15) == 0) continue;
        const int64_t t = (int64_t)c * 256 + tid;
        uint32_t key = 0;
        if (t < L && !forced_bit(forced, t)) key = f32_key(score_token(w[x], lb, T));
        push_cands(key != 0 && key >= tau, key, (uint32_t)t);
      }
    }
    __syncthreads();
    const int nc = ms->ncand;
    fallback = (nc > a.cap) || (nc < keff);
    if (!fallback) {
      // ---------------- C: exact k-th key among the candidates
      if (tid == 0) ms->rem_sel = keff;
      uint32_t prefix = 0, pmask = 0;
      for (int shift = 24; shift >= 0; shift -= 8) {
        hist[tid] = 0;
        __syncthreads();
        for (int i0 = 0; i0 < nc; i0 += DT) {
          const int i = i0 + tid;
          const uint32_t key = i < nc ? cand[2 * i] : 0u;
          hist_add(hist, (i < nc && (key & pmask) == prefix) ? (int)((key >> shift) & 255) : -1);
        }
        __syncthreads();
        pick_digit(hist, ms);
        __syncthreads();
        prefix |= (uint32_t)ms->digit << shift;
        pmask |= 0xFFu << shift;
        if (tid == 0) ms->rem_sel -= ms->cnt_above;
        __syncthreads();
      }
      kstar = prefix;
      need_eq = ms->rem_sel;
      // bitmaps live in R0 (the pair table is dead now)
      gt = reinterpret_cast<uint32_t*>(T);
      eq = gt + W;
      for (int i = tid; i < 2 * W; i += DT) gt[i] = 0u;
      __syncthreads();
      for (int i = tid; i < nc; i += DT) {
        const uint32_t key = cand[2 * i], t = cand[2 * i + 1];
        if (key > kstar) atomicOr(&gt[t >> 5], 1u << (t & 31));
        else if (key == kstar) atomicOr(&eq[t >> 5], 1u << (t & 31));
      }
      __syncthreads();
    }
  }
  if (fallback) {
    // ---------------- exact multi-pass radix select by rescoring (rare)
    if (tid == 0) { ms->rem_sel = keff; ms->fb = 1; }
    uint32_t prefix = 0, pmask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      hist[tid] = 0;
      __syncthreads();
      for (int c = 0; c < nchunks; ++c) {
        const int64_t t = (int64_t)c * 256 + tid;
        uint32_t key = 0;
        if (t < L && !forced_bit(forced, t)) key = f32_key(score_token(__ldg(signs + t), lb, T));
        hist_add(hist, (key != 0 && (key & pmask) == prefix) ? (int)((key >> shift) & 255) : -1);
      }
      __syncthreads();
      pick_digit(hist, ms);
      __syncthreads();
      prefix |= (uint32_t)ms->digit << shift;
      pmask |= 0xFFu << shift;
      if (tid == 0) ms->rem_sel -= ms->cnt_above;
      __syncthreads();
    }
    kstar = prefix;
    need_eq = ms->rem_sel;
    gt = cand;                       // candidates are dead; bitmaps go there
    eq = gt + W;
    for (int i = tid; i < 2 * W; i += DT) gt[i] = 0u;
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
      const int64_t t = (int64_t)c * 256 + tid;
      uint32_t key = 0;
      if (t < L && !forced_bit(forced, t)) key = f32_key(score_token(__ldg(signs + t), lb, T));
      if (key != 0 && key > kstar) atomicOr(&gt[t >> 5], 1u << (t & 31));
      else if (key != 0 && key == kstar) atomicOr(&eq[t >> 5], 1u << (t & 31));
    }
    __syncthreads();
  }

  // ---------------- ordered scan: dynamic list (smem) + sorted selection (global)
  int32_t* dyn = reinterpret_cast<int32_t*>(sm + a.off_lists);
  {
    const int per = (W + DT - 1) / DT;
    const int w0 = tid * per, w1 = min(W, w0 + per);
    // pass 1: eq bits before this thread
    int my_eq = 0;
    if (mode >= 2) for (int x = w0; x < w1; ++x) my_eq += __popc(eq[x]);
    int eq_before, dummy, t1, t2;
    block_exscan2(my_eq, 0, eq_before, dummy, t1, t2, ms->wsum);
    // pass 2: counts
    int nd = 0, nsl = 0;
    int eb = eq_before;
    for (int x = w0; x < w1; ++x) {
      uint32_t d;
      if (mode == 0) d = 0u;
      else if (mode == 1) {
        d = ~forced[x];
        if (x == W - 1 && (L & 31)) d &= (1u << (L & 31)) - 1u;
      } else {
        uint32_t e = eq[x];
        int take = min(max(need_eq - eb, 0), __popc(e));
        eb += __popc(e);
        while (__popc(e) > take) e &= ~(1u << (31 - __clz(e)));
        d = gt[x] | e;
      }
      nd += __popc(d);
      nsl += __popc(d | forced[x]);
    }
    int dpos, spos, dtot, stot;
    block_exscan2(nd, nsl, dpos, spos, dtot, stot, ms->wsum);
    eb = eq_before;
    for (int x = w0; x < w1; ++x) {
      uint32_t d;
      if (mode == 0) d = 0u;
      else if (mode == 1) {
        d = ~forced[x];
        if (x == W - 1 && (L & 31)) d &= (1u << (L & 31)) - 1u;
      } else {
        uint32_t e = eq[x];
        int take = min(max(need_eq - eb, 0), __popc(e));
        eb += __popc(e);
        while (__popc(e) > take) e &= ~(1u << (31 - __clz(e)));
        d = gt[x] | e;
      }
      uint32_t sb = d | forced[x];
      while (d) { int b = __ffs(d) - 1; d &= d - 1; dyn[dpos++] = x * 32 + b; }
      if (a.sel) {
        while (sb) { int b = __ffs(sb) - 1; sb &= sb - 1; a.sel[u * a.sel_stride + spos++] = x * 32 + b; }
      }
    }
    if (a.sel && tid < R) a.sel[u * a.sel_stride + stot + tid] = (int32_t)(L + tid);
    if (tid == 0) {
      ms->total = dtot;
      if (a.sel_count) a.sel_count[u] = stot + R;
      if (a.diag) a.diag[u] = (mode & 3) | (ms->fb ? 4 : 0);
    }
  }
  __syncthreads();
  const int ndyn = ms->total;

  // ---------------- D: sparse attention over forced rows + dynamic rows
  const int g = lane >> 2, t4 = lane & 3;
  // q~ = q * alpha-hat as fp16 A fragments (row g = head g; rows >= Gq are zero)
  uint32_t qa[8][2];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int d = 16 * s + 2 * t4 + 8 * e;
      float x0 = 0.f, x1 = 0.f;
      if (g < Gq) {
        x0 = qs[g * FD + d] * ahat[d];
        x1 = qs[g * FD + d + 1] * ahat[d + 1];
      }
      qa[s][e] = h2u(__floats2half2_rn(x0, x1));
    }
  }
  const float sc = 1.4426950408889634f * rsqrtf((float)FD);
  float o[8][4];
#pragma unroll
  for (int m = 0; m < 8; ++m) o[m][0] = o[m][1] = o[m][2] = o[m][3] = 0.f;
  float mrun = -INFINITY, lrun = 0.f;   // for head g (shared by the quad)

  const int nf = S + R;
  const int nbf = (nf + 15) >> 4, nbd = (ndyn + 15) >> 4;
  const uint8_t* recs = a.recs + u * L * FREC;

  for (int blk = warp; blk < nbf + nbd; blk += DW) {
    uint32_t kb[2][8][2];     // K^ B fragments for tokens g (nt=0) and g+8 (nt=1)
    uint32_t va[8][4];        // V^T A fragments
    bool valid[2][2];         // this thread's score columns: [nt][lo/hi]
    if (blk < nbf) {
      // forced rows (fp32 K', V): sinks then recents
      const int base = blk * 16;
      auto rowk = [&](int f) -> const float* {
        return f < S ? a.sink_k + (u * S + f) * FD : a.rec_k + (u * a.rcap + (f - S)) * FD;
      };
      auto rowv = [&](int f) -> const float* {
        return f < S ? a.sink_v + (u * S + f) * FD : a.rec_v + (u * a.rcap + (f - S)) * FD;
      };
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int f = min(base + g + 8 * nt, nf - 1);
        const float* kr = rowk(f);
#pragma unroll
        for (int s = 0; s < 8; ++s)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = 16 * s + 2 * t4 + 8 * e;
            const float2 kk = *reinterpret_cast<const float2*>(kr + d);
            kb[nt][s][e] = h2u(__floats2half2_rn(kk.x / ahat[d], kk.y / ahat[d + 1]));
          }
        valid[nt][0] = base + 2 * t4 + 8 * nt < nf;
        valid[nt][1] = base + 2 * t4 + 1 + 8 * nt < nf;
      }
      const float* vr[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) vr[x] = rowv(min(base + 2 * t4 + (x & 1) + 8 * (x >> 1), nf - 1));
#pragma unroll
      for (int m = 0; m < 8; ++m)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int d = 16 * m + g + 8 * (r & 1), pr = r >> 1;
          va[m][r] = h2u(__floats2half2_rn(vr[2 * pr][d], vr[2 * pr + 1][d]));
        }
    } else {
      // dynamic rows: dequantise 2-bit records
      const int base = (blk - nbf) * 16;
      int tk[2], tv[4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) tk[nt] = dyn[min(base + g + 8 * nt, ndyn - 1)];
#pragma unroll
      for (int x = 0; x < 4; ++x) tv[x] = dyn[min(base + 2 * t4 + (x & 1) + 8 * (x >> 1), ndyn - 1)];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        valid[nt][0] = base + 2 * t4 + 8 * nt < ndyn;
        valid[nt][1] = base + 2 * t4 + 1 + 8 * nt < ndyn;
      }
      // loads
      uint2 kw[2]; uint4 kp[2]; uint32_t ks[2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const uint8_t* r = recs + (int64_t)tk[nt] * FREC;
        kw[nt] = __ldg(reinterpret_cast<const uint2*>(r + R_KPAY) + t4);
        kp[nt] = __ldg(reinterpret_cast<const uint4*>(r + R_KPAR));
        ks[nt] = __ldg(reinterpret_cast<const uint32_t*>(r + R_KSGN) + t4);
      }
      uint32_t vw[4]; uint4 vp[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint8_t* r = recs + (int64_t)tv[x] * FREC;
        vw[x] = __ldg(reinterpret_cast<const uint32_t*>(r + R_VPAY) + g);
        vp[x] = __ldg(reinterpret_cast<const uint4*>(r + R_VPAR));
      }
      const uint32_t magic[4] = {0x64006400u, 0x5C005C00u, 0x54005400u, 0x4C004C00u};
      // K^ = sign * (qs*c + zp)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const uint32_t par[4] = {kp[nt].x, kp[nt].y, kp[nt].z, kp[nt].w};
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const uint32_t wd = uu ? kw[nt].y : kw[nt].x;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int s = 4 * uu + (i >> 1), e = i & 1, grp = s >> 1;
            const uint32_t src = i < 4 ? wd : (wd >> 8);
            const int ii = i & 3;
            const uint32_t x = lop3_and_or(src, 0x00030003u << (2 * ii), magic[ii]);
            const __half2 c = __hsub2(u2h(x), u2h(magic[ii]));
            const __half2 qs2 = u2h(prmt(par[grp], par[grp], 0x1010u));
            const __half2 zp2 = u2h(prmt(par[grp], par[grp], 0x3232u));
            const uint32_t v = h2u(__hfma2(c, qs2, zp2));
            const int P = 8 * uu + i;
            kb[nt][s][e] = lop3_xor_and(v, ks[nt] << (15 - P), 0x80008000u);
          }
        }
      }
      // V^T fragments: pairs (2t4, 2t4+1) and (2t4+8, 2t4+9)
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const uint32_t wa = vw[2 * pr], wb = vw[2 * pr + 1];
        const uint32_t pa[4] = {vp[2 * pr].x, vp[2 * pr].y, vp[2 * pr].z, vp[2 * pr].w};
        const uint32_t pb[4] = {vp[2 * pr + 1].x, vp[2 * pr + 1].y, vp[2 * pr + 1].z, vp[2 * pr + 1].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t xj = prmt(wa, wb, (uint32_t)(j | (j << 4) | ((4 + j) << 8) | ((4 + j) << 12)));
          const __half2 qs2 = u2h(prmt(pa[j], pb[j], 0x5410u));
          const __half2 zp2 = u2h(prmt(pa[j], pb[j], 0x7632u));
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int m = 2 * j + (ii >> 1), e = ii & 1;
            const uint32_t x = lop3_and_or(xj, 0x00030003u << (2 * ii), magic[ii]);
            const __half2 c = __hsub2(u2h(x), u2h(magic[ii]));
            va[m][2 * pr + e] = h2u(__hfma2(c, qs2, zp2));
          }
        }
      }
    }
    // ---- scores S^T[h][tok] = q~ . K^
    float sacc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) mma16816(sacc[nt], qa[s][0], 0u, qa[s][1], 0u, kb[nt][s][0], kb[nt][s][1]);
    }
    // ---- online softmax for head g over this block's 16 tokens
    float x[4];
    x[0] = valid[0][0] ? sacc[0][0] * sc : -INFINITY;
    x[1] = valid[0][1] ? sacc[0][1] * sc : -INFINITY;
    x[2] = valid[1][0] ? sacc[1][0] * sc : -INFINITY;
    x[3] = valid[1][1] ? sacc[1][1] * sc : -INFINITY;
    float bm = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
    const float mnew = fmaxf(mrun, bm);
    const float fac = exp2f(mrun - mnew);
    mrun = mnew;
    __half2 p01 = __floats2half2_rn(exp2f(x[0] - mnew), exp2f(x[1] - mnew));
    __half2 p23 = __floats2half2_rn(exp2f(x[2] - mnew), exp2f(x[3] - mnew));
    const float2 f01 = __half22float2(p01), f23 = __half22float2(p23);
    lrun = lrun * fac + ((f01.x + f01.y) + (f23.x + f23.y));
    // rescale O columns h = 2t4, 2t4+1 by their heads' factors (held by quads g = 2t4, 2t4+1)
    const float fa = __shfl_sync(0xffffffffu, fac, 8 * t4);
    const float fb = __shfl_sync(0xffffffffu, fac, 8 * t4 + 4);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      o[m][0] *= fa; o[m][1] *= fb; o[m][2] *= fa; o[m][3] *= fb;
      mma16816(o[m], va[m][0], va[m][1], va[m][2], va[m][3], h2u(p01), h2u(p23));
    }
  }

  // ---------------- merge the 8 warp partials (fixed order)
  __syncthreads();
  float* part = reinterpret_cast<float*>(cand);           // [DW][Gq][128]
  float* pm = part + DW * Gq * FD;                         // [DW][Gq]
  float* pl = pm + DW * Gq;                                // [DW][Gq]
  {
    float l = lrun;
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (t4 == 0 && g < Gq) { pm[warp * Gq + g] = mrun; pl[warp * Gq + g] = l; }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int h0 = 2 * t4, h1 = 2 * t4 + 1, d0 = 16 * m + g, d1 = d0 + 8;
      if (h0 < Gq) { part[(warp * Gq + h0) * FD + d0] = o[m][0]; part[(warp * Gq + h0) * FD + d1] = o[m][2]; }
      if (h1 < Gq) { part[(warp * Gq + h1) * FD + d0] = o[m][1]; part[(warp * Gq + h1) * FD + d1] = o[m][3]; }
    }
  }
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
    a.out[(u * Gq + h) * FD + d] = num / den;
    if (a.lse && d == 0) a.lse[u * Gq + h] = (M + log2f(den)) * 0.6931471805599453f;
  }
}

// ---------------------------------------------------------------- scores only (tests / API)
__global__ void score_fast_kernel(const uint8_t* __restrict__ signs_, const float* __restrict__ cent32,
                                  const float* __restrict__ q, int Gq, int64_t L, float* __restrict__ out) {
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
    const float4 c = reinterpret_cast<const float4*>(C)[e];
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
  const uint32_t lb = (uint32_t)(64 * ((lane >> 4) & 1) + 4 * (lane & 15));
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + tid; t < L; t += (int64_t)gridDim.x * blockDim.x)
    out[u * L + t] = score_token(__ldg(signs + t), lb, T);
}

// ---------------------------------------------------------------- host side

static int align16(int x) { return (x + 15) & ~15; }

DecodeLayout decode_layout(int64_t L, int k, int S, int Gq, int cap) {
  DecodeLayout d{};
  const int W = (int)((L + 31) / 32);
  const int nchunks = (int)((L + 255) / 256);
  d.nsamp = ((nchunks + 15) / 16) * 256;
  const int keff = (int)std::min<int64_t>(k, L - S);
  // R0: pair table, later gt/eq bitmaps (fast path) followed by the dynamic list
  int r0 = std::max(TBL_BYTES, align16(2 * W * 4) + align16(std::max(keff, 1) * 4));
  // fallback path puts the bitmaps into R1 and the list at R0 start
  int r1 = std::max(cap * 8, 2 * W * 4);
  r1 = std::max(r1, DW * Gq * (FD + 2) * 4);            // attention partials
  int off = align16(r0);
  d.off_lists = align16(2 * W * 4);                     // dynamic list after fast-path bitmaps
  d.off_cand = off;
  // sample keys: alias the tail of R1 when that cannot collide with candidate writes
  if ((int64_t)d.nsamp * 12 <= (int64_t)r1 * 1) {
    d.off_samp = off + r1 - d.nsamp * 4;
    off += align16(r1);
  } else {
    off += align16(r1);
    d.off_samp = off;
    off += align16(d.nsamp * 4);
  }
  d.off_forced = off;
  off += align16(W * 4);
  d.off_misc = off;
  off += 256 + (8 * FD + 512 + FD + FD + FD + 256) * 4;
  d.total = align16(off);
  return d;
}

cudaError_t launch_decode(const uint8_t* signs, const uint8_t* recs, const float* cent32,
                          const float* alpha32, const int32_t* sink_idx, int S, const float* sink_k,
                          const float* sink_v, const float* rec_k, const float* rec_v, int64_t rcap, int R,
                          const float* q, int64_t U, int64_t L, int Gq, int k, int cap, float* out,
                          float* lse, int32_t* sel, int sel_stride, int32_t* sel_count, int32_t* diag,
                          cudaStream_t st, int* smem_out) {
  DecodeLayout d = decode_layout(L, k, S, Gq, cap);
  if (smem_out) *smem_out = d.total;
  DecodeArgs a{signs, recs, cent32, alpha32, sink_idx, sink_k, sink_v, rec_k, rec_v, q, out, lse, sel,
               sel_count, diag, L, rcap, S, R, Gq, k, cap, sel_stride, d.nsamp,
               d.off_cand, d.off_samp, d.off_forced, d.off_misc, d.off_lists};
  cudaError_t e = cudaFuncSetAttribute(decode_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, d.total);
  if (e != cudaSuccess) return e;
  decode_step_kernel<<<(unsigned)U, DT, d.total, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_score_fast(const uint8_t* signs, const float* cent32, const float* q, int Gq,
                              int64_t U, int64_t L, float* out, cudaStream_t st) {
  const int bx = (int)std::min<int64_t>(64, (L + 255) / 256);
  cudaError_t e = cudaFuncSetAttribute(score_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TBL_BYTES);
  if (e != cudaSuccess) return e;
  score_fast_kernel<<<dim3(bx, (unsigned)U), 256, TBL_BYTES, st>>>(signs, cent32, q, Gq, L, out);
  return cudaGetLastError();
}

}  // namespace sikv
