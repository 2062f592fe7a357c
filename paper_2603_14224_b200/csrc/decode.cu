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

__device__ long long* g_prof = nullptr;   // optional per-unit phase clocks (debug / profiling)

constexpr int NB = 8;                     // chunks (of 256 tokens) scored per thread per batch
constexpr int STAGE_BYTES = 16 * FREC;    // one 16-token block of records
constexpr int MAX_SAMPLE_CHUNKS = 8;

struct DecodeArgs {
  const uint8_t* signs;     // [U][L][16] rotated sign plane
  const uint8_t* recs;      // [U][L][128] records
  const float* cent32;      // [U][32][16][4]
  const float* alpha32;     // [U][128]
  const int32_t* sink_idx;  // [U][S] sorted, unique, < L
  const uint32_t* ffrag;    // [U][fblocks][2][32 lanes][32 words] forced rows as fp16 fragments
  const float* q;           // [U][Gq][128]
  float* out;               // [U][Gq][128]
  float* lse;               // [U][Gq] natural-log sum of exp(logits), nullable
  int32_t* sel;             // [U][sel_stride], nullable
  int32_t* sel_count;       // [U], nullable
  int32_t* diag;            // [U], nullable
  int64_t L;
  int fblocks;
  int S, R, Gq, k, capw, sel_stride;
  // shared-memory layout (byte offsets)
  int off_cand, off_forced, off_misc, off_bits, off_dyn, off_stage;
};

// ---------------------------------------------------------------- scoring
// score of the token whose 16-byte rotated sign record is w; lb = byte offset of this
// lane's first column (64*half + 4*j); T = pair table (row stride 256 B).  Pairs are
// summed left to right starting at pair (t mod 16) — the order oracle/restate32.py states.
__device__ __forceinline__ float score_token(const uint4 w, uint32_t lb, const char* T) {
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t off = prmt(ww[i >> 2], lb, 0x5504u | ((uint32_t)(i & 3) << 4));
    const float v = *reinterpret_cast<const float*>(T + off + 4 * i);
    s = (i == 0) ? v : __fadd_rn(s, v);
  }
  return s;
}

// NB tokens at once: the 16-step chains of different tokens interleave, hiding FADD latency
template <int N>
__device__ __forceinline__ void score_batch(const uint4 (&w)[N], uint32_t lb, const char* T, float (&s)[N]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int x = 0; x < N; ++x) {
      const uint32_t wd = (i >> 2) == 0 ? w[x].x : (i >> 2) == 1 ? w[x].y : (i >> 2) == 2 ? w[x].z : w[x].w;
      const uint32_t off = prmt(wd, lb, 0x5504u | ((uint32_t)(i & 3) << 4));
      const float v = *reinterpret_cast<const float*>(T + off + 4 * i);
      s[x] = (i == 0) ? v : __fadd_rn(s[x], v);
    }
  }
}

__device__ __forceinline__ bool forced_bit(const uint32_t* fb, int64_t t) {
  return (fb[t >> 5] >> (t & 31)) & 1u;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// stage the 16 records of one dynamic block into shared memory, 16-byte chunk k of token j
// stored at chunk k ^ (j & 7) so the fragment reads below are bank-conflict free
__device__ __forceinline__ void stage_block(char* buf, const uint8_t* recs, const int32_t* dyn, int base,
                                            int ndyn, int lane) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int c = lane + 32 * r, j = c >> 3, kk = c & 7;
    const int t = dyn[min(base + j, ndyn - 1)];
    cp_async16(buf + j * FREC + 16 * (kk ^ (j & 7)), recs + (int64_t)t * FREC + 16 * kk);
  }
}
__device__ __forceinline__ const char* chunk(const char* buf, int j, int kk) {
  return buf + j * FREC + 16 * (kk ^ (j & 7));
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(DT, 2) decode_step_kernel(DecodeArgs a) {
  extern __shared__ __align__(128) char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t u = blockIdx.x;
  const int64_t L = a.L;
  const int W = (int)((L + 31) >> 5);
  char* T = sm;                                                   // R0: pair table
  uint32_t* cand = reinterpret_cast<uint32_t*>(sm + a.off_cand);  // R1: per-warp (x, t) segments
  uint32_t* forced = reinterpret_cast<uint32_t*>(sm + a.off_forced);
  Misc* ms = reinterpret_cast<Misc*>(sm + a.off_misc);
  float* qs = reinterpret_cast<float*>(sm + a.off_misc + 256);    // [Gq][128]
  float* lut = qs + 8 * FD;                                       // [32][16]
  float* qbar = lut + 512;                                        // [128]
  float* inva = qbar + FD;                                        // [128] 1 / alpha-hat
  float* ahat = inva + FD;                                        // [128] alpha-hat

  const uint4* signs = reinterpret_cast<const uint4*>(a.signs + u * L * FSIGN);
  const int S = a.S, R = a.R, Gq = a.Gq, capw = a.capw;

  // ---------------- A: queries, LUT, pair table, forced bitmap
  for (int i = tid; i < Gq * FD; i += DT) qs[i] = a.q[u * Gq * FD + i];
  for (int i = tid; i < W; i += DT) forced[i] = 0u;
  long long* prof = g_prof ? g_prof + u * 12 : nullptr;
#define PROF(i) do { if (prof && tid == 0) prof[i] = clock64(); } while (0)
  PROF(0);
  // selection mode and sample geometry first, so the sample's HBM loads overlap the setup
  const int64_t ncand_all = L - S;
  const int keff = (int)((int64_t)a.k < ncand_all ? (int64_t)a.k : ncand_all);
  const int nchunks = (int)((L + 255) >> 8);
  // selection modes: 0 nothing dynamic, 1 every candidate, 2 all candidates fit (tau = -inf),
  // 3 sampled threshold
  int mode;
  if (keff == 0) mode = 0;
  else if (keff == ncand_all) mode = 1;
  else if ((int64_t)nchunks * 32 <= (int64_t)capw) mode = 2;   // every warp's tokens fit its segment
  else mode = 3;
  const int sstride = mode == 3 ? max(16, (nchunks + MAX_SAMPLE_CHUNKS - 1) / MAX_SAMPLE_CHUNKS) : 1;
  const int nsc = mode == 3 ? (nchunks + sstride - 1) / sstride : 0;
  uint4 wsamp[MAX_SAMPLE_CHUNKS];
#pragma unroll
  for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
    const int64_t t = (int64_t)x * sstride * 256 + tid;
    wsamp[x] = (x < nsc && t < L) ? __ldg(signs + t) : make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) { ms->fb = 0; ms->maxx = 0; ms->bad = 0; }
  __syncthreads();
  for (int j = tid; j < S; j += DT) {
    const int t = a.sink_idx[u * S + j];
    atomicOr(&forced[t >> 5], 1u << (t & 31));
  }
  if (tid < FD) {
    float s = qs[tid];
    for (int h = 1; h < Gq; ++h) s = __fadd_rn(s, qs[h * FD + tid]);
    qbar[tid] = s;
    const float al = a.alpha32[u * FD + tid];
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
    row[p] = v; row[p + 16] = v; row[p + 32] = v;
  }
  __syncthreads();

  const int64_t flim = S > 0 ? (int64_t)a.sink_idx[u * S + S - 1] + 1 : 0;   // sinks are sorted
  const uint32_t lb = (uint32_t)(64 * ((lane >> 4) & 1) + 4 * (lane & 15));

  uint32_t* gt = reinterpret_cast<uint32_t*>(sm + a.off_bits);
  uint32_t* eq = gt + W;
  int* hist = reinterpret_cast<int*>(sm);          // fast path: R0 front once scoring is done
  uint32_t kstar = 0;
  int need_eq = 0;

  // per-warp candidate segment: entries (x = key - tau, t)
  uint32_t* seg = cand + 2 * warp * capw;
  int wc = 0;                  // warp-uniform fill count
  uint32_t mx = 0;             // per-thread max x
  // warp-compacted append of this thread's flagged tokens (bit x of `bits` <-> sv[x], token
  // t0 + 256 x); one warp scan per batch instead of one ballot per token
  auto push_batch = [&](uint32_t bits, const float* sv, int nb, int t0, uint32_t tau) {
    const int cnt = __popc(bits);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int pos = wc + inc - cnt;
    wc += __shfl_sync(0xffffffffu, inc, 31);
    while (bits) {
      const int x = __ffs(bits) - 1;
      bits &= bits - 1;
      float v = sv[0];
#pragma unroll
      for (int y = 1; y < NB; ++y) v = (x == y) ? sv[y] : v;
      const uint32_t xk = f32_key(v) - tau;
      if (pos < capw) { seg[2 * pos] = xk; seg[2 * pos + 1] = (uint32_t)(t0 + 256 * x); }
      mx = max(mx, xk);
      ++pos;
    }
  };

  bool fallback = false;
  if (mode >= 2) {
    uint32_t tau = 1;
    if (mode == 3) {
      PROF(1);
      // ---------------- B1: score the sample chunks (<= 8 per thread, kept in registers)
      uint32_t sk[MAX_SAMPLE_CHUNKS];
      float sv[MAX_SAMPLE_CHUNKS];
      score_batch(wsamp, lb, T, sv);
      int nv = 0;
      uint32_t smax = 0, smin = 0xFFFFFFFFu;
#pragma unroll
      for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
        const int64_t t = (int64_t)x * sstride * 256 + tid;
        uint32_t key = 0;
        if (x < nsc && t < L && !(t < flim && forced_bit(forced, t))) key = f32_key(sv[x]);
        sk[x] = key;
        nv += key != 0;
        smax = max(smax, key);
        if (key) smin = min(smin, key);
      }
      nv = warp_sum(nv);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
      }
      // threshold histogram: 256 value-linear bins over [smin, smax] of the sample
      int* th = reinterpret_cast<int*>(cand);                  // [256] counts
      uint32_t* tmin = reinterpret_cast<uint32_t*>(cand) + 256; // [256] min key per bin
      for (int i = tid; i < 256; i += DT) { th[i] = 0; tmin[i] = 0xFFFFFFFFu; }
      if (tid == 0) { ms->nsv = 0; ms->tau = 0xFFFFFFFFu; }
      __syncthreads();
      if (lane == 0) { atomicAdd(&ms->nsv, nv); atomicMax(&ms->maxx, smax); atomicMin(&ms->tau, smin); }
      __syncthreads();
      const int nsv = ms->nsv;
      const double e = (double)keff * (double)nsv / (double)ncand_all;
      int r = (int)ceil(e + 4.0 * sqrt(e) + 16.0);
      r = min(r, nsv);
      if (r >= 1) {
        const uint32_t kmx = ms->maxx, kmn = ms->tau;
        auto unkey = [](uint32_t k2) {
          return __uint_as_float((k2 & 0x80000000u) ? (k2 & 0x7FFFFFFFu) : ~k2);
        };
        const float fmn = unkey(kmn), fmx = unkey(kmx);
        const float scale = fmx > fmn ? 256.0f / (fmx - fmn) : 0.f;
#pragma unroll
        for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
          if (sk[x]) {
            const int b = min(255, (int)((unkey(sk[x]) - fmn) * scale));
            atomicAdd(&th[b], 1);
            atomicMin(&tmin[b], sk[x]);
          }
        }
        __syncthreads();
        if (warp == 0) {
          int loc[8], s8 = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) { loc[i] = th[255 - 8 * lane - i]; s8 += loc[i]; }
          int inc = s8;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
          }
          int c = inc - s8;
          if (c < r && r <= inc) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (c < r && r <= c + loc[i]) ms->digit = 255 - 8 * lane - i;
              c += loc[i];
            }
          }
        }
        __syncthreads();
        tau = tmin[ms->digit];          // smallest sample key in the boundary bin
      }
      __syncthreads();
      if (tid == 0) ms->maxx = 0;
      __syncthreads();
      {
        uint32_t bits = 0;
#pragma unroll
        for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x)
          if (x < nsc && sk[x] != 0 && sk[x] >= tau) bits |= 1u << x;
        int cnt = __popc(bits), inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += v;
        }
        int pos = wc + inc - cnt;
        wc += __shfl_sync(0xffffffffu, inc, 31);
#pragma unroll
        for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
          if ((bits >> x) & 1u) {
            const uint32_t xk = sk[x] - tau;
            if (pos < capw) { seg[2 * pos] = xk; seg[2 * pos + 1] = (uint32_t)(x * sstride * 256 + tid); }
            mx = max(mx, xk);
            ++pos;
          }
        }
      }
    }
    PROF(2);
    // ---------------- B2: score everything else, keep score >= tau (compared as floats)
    float tauf;
    {
      const uint32_t k2 = tau;
      tauf = mode == 2 ? -INFINITY : __uint_as_float((k2 & 0x80000000u) ? (k2 & 0x7FFFFFFFu) : ~k2);
    }
    const int Li = (int)L;
    int next_s = mode == 3 ? 0 : 0x7fffffff;      // next sample chunk (already scored in B1)
    const int end_s = nsc * sstride;
    for (int c0 = 0; c0 < nchunks; c0 += NB) {
      int xs = -1;                  // the (at most one, sstride >= 16 > NB) sample chunk here
      if (next_s < c0 + NB && next_s < end_s) { xs = next_s - c0; next_s += sstride; }
      const int t0 = c0 * 256 + tid;
      const bool full = (c0 + NB) * 256 <= Li;
      uint4 w[NB];
      if (full) {
#pragma unroll
        for (int x = 0; x < NB; ++x) w[x] = __ldg(signs + t0 + 256 * x);
      } else {
#pragma unroll
        for (int x = 0; x < NB; ++x) w[x] = t0 + 256 * x < Li ? __ldg(signs + t0 + 256 * x) : make_uint4(0, 0, 0, 0);
      }
      float sv[NB];
      score_batch(w, lb, T, sv);
      uint32_t bits = 0;
#pragma unroll
      for (int x = 0; x < NB; ++x)
        if (sv[x] >= tauf) bits |= 1u << x;
      if (xs >= 0) bits &= ~(1u << xs);
      if (!full) bits &= (Li - t0 > 0) ? ((Li - t0 + 255) / 256 >= NB ? 0xFFu : ((1u << ((Li - t0 + 255) / 256)) - 1u)) : 0u;
      if (c0 * 256 < flim) {
#pragma unroll
        for (int x = 0; x < NB; ++x)
          if (t0 + 256 * x < Li && forced_bit(forced, t0 + 256 * x)) bits &= ~(1u << x);
      }
      push_batch(bits, sv, NB, t0, tau);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) { ms->wcnt[warp] = wc; atomicMax(&ms->maxx, mx); if (wc > capw) ms->bad = 1; }
    __syncthreads();
    int total = 0;
    for (int w2 = 0; w2 < DW; ++w2) total += ms->wcnt[w2];
    fallback = ms->bad || total < keff;
    if (!fallback) {
      PROF(3);
      // ---------------- C: exact k-th key among the candidates (pair table is dead now)
      const int n = wc;   // this warp's segment
      uint32_t xk;
      radix_kth([&](auto f) {
        for (int i = lane; i < n; i += 32) f(seg[2 * i]);
      }, ms->maxx, keff, hist, ms, xk, need_eq);
      kstar = xk + tau;
      for (int i = tid; i < 2 * W; i += DT) gt[i] = 0u;
      if (tid == 0) ms->nsv = 0;
      __syncthreads();
      for (int i = lane; i < n; i += 32) {
        const uint32_t x = seg[2 * i], t = seg[2 * i + 1];
        if (x > xk) atomicOr(&gt[t >> 5], 1u << (t & 31));
        else if (x == xk) { atomicOr(&eq[t >> 5], 1u << (t & 31)); atomicAdd(&ms->nsv, 1); }
      }
      __syncthreads();
    }
  }
  if (fallback) {
    // ---------------- exact multi-pass radix select by rescoring (rare)
    if (tid == 0) ms->fb = 1;
    int* fh = reinterpret_cast<int*>(cand);        // candidates are void; hist + bitmaps go there
    uint32_t* fgt = reinterpret_cast<uint32_t*>(sm + a.off_cand + NBIN * 4);
    uint32_t* feq = fgt + W;
    radix_kth([&](auto f) {
      for (int c = 0; c < nchunks; ++c) {
        const int64_t t = (int64_t)c * 256 + tid;
        if (t < L && !forced_bit(forced, t)) f(f32_key(score_token(__ldg(signs + t), lb, T)));
      }
    }, 0xFFFFFFFFu, keff, fh, ms, kstar, need_eq);
    for (int i = tid; i < 2 * W; i += DT) fgt[i] = 0u;
    if (tid == 0) ms->nsv = 0;
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
      const int64_t t = (int64_t)c * 256 + tid;
      if (t < L && !forced_bit(forced, t)) {
        const uint32_t key = f32_key(score_token(__ldg(signs + t), lb, T));
        if (key > kstar) atomicOr(&fgt[t >> 5], 1u << (t & 31));
        else if (key == kstar) { atomicOr(&feq[t >> 5], 1u << (t & 31)); atomicAdd(&ms->nsv, 1); }
      }
    }
    __syncthreads();
    // move the bitmaps to their fast-path home (the pair table is dead now)
    for (int i = tid; i < 2 * W; i += DT) gt[i] = fgt[i];
    __syncthreads();
  }

  PROF(4);
  // ---------------- ordered scan: dynamic list (smem) + sorted selection (global)
  int32_t* dyn = reinterpret_cast<int32_t*>(sm + a.off_dyn);
  {
    const int per = (W + DT - 1) / DT;
    const int w0 = tid * per, w1 = min(W, w0 + per);
    // ties at the k-th key: keep the lowest-index need_eq of them (prefix over the eq
    // bitmap); when every tie is taken (the usual case) no prefix is needed
    const bool all_eq = mode < 2 || ms->nsv == need_eq;
    int eq_before = 0;
    if (!all_eq) {
      int my_eq = 0;
      for (int x = w0; x < w1; ++x) my_eq += __popc(eq[x]);
      int dummy, t1, t2;
      block_exscan2(my_eq, 0, eq_before, dummy, t1, t2, ms->wsum);
    }
    auto dbits = [&](int x, int& eb) -> uint32_t {
      if (mode == 0) return 0u;
      if (mode == 1) {
        uint32_t d = ~forced[x];
        if (x == W - 1 && (L & 31)) d &= (1u << (L & 31)) - 1u;
        return d;
      }
      uint32_t e = eq[x];
      if (!all_eq) {
        const int take = min(max(need_eq - eb, 0), __popc(e));
        eb += __popc(e);
        while (__popc(e) > take) e &= ~(1u << (31 - __clz(e)));
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
    block_exscan2(nd, nsl, dpos, spos, dtot, stot, ms->wsum);
    eb = eq_before;
    for (int x = w0; x < w1; ++x) {
      uint32_t d = dbits(x, eb);
      uint32_t sb = d | forced[x];
      while (d) { const int b = __ffs(d) - 1; d &= d - 1; dyn[dpos++] = x * 32 + b; }
      if (a.sel)
        while (sb) { const int b = __ffs(sb) - 1; sb &= sb - 1; a.sel[u * a.sel_stride + spos++] = x * 32 + b; }
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

  PROF(5);
  // ---------------- D: sparse attention over forced rows + dynamic rows
  const int g = lane >> 2, t4 = lane & 3;
  uint32_t qa[8][2];       // q~ = q * alpha-hat, fp16 A fragments (row g = head g)
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int d = 16 * s + 2 * t4 + 8 * e;
      float x0 = 0.f, x1 = 0.f;
      if (g < Gq) { x0 = qs[g * FD + d] * ahat[d]; x1 = qs[g * FD + d + 1] * ahat[d + 1]; }
      qa[s][e] = h2u(__floats2half2_rn(x0, x1));
    }
  const float sc = 1.4426950408889634f * rsqrtf((float)FD);
  float o[8][4];
#pragma unroll
  for (int m = 0; m < 8; ++m) o[m][0] = o[m][1] = o[m][2] = o[m][3] = 0.f;
  float mrun = -INFINITY, lrun = 0.f;   // head g, shared by the quad

  const int nf = S + R;
  const int nbf = (nf + 15) >> 4, nbd = (ndyn + 15) >> 4;
  const uint8_t* recs = a.recs + u * L * FREC;
  char* stage = sm + a.off_stage + warp * 2 * STAGE_BYTES;
  const uint32_t magic[4] = {0x64006400u, 0x5C005C00u, 0x54005400u, 0x4C004C00u};

  // online softmax update + P V for one block, given the block's scores and V fragments source
  auto softmax_pv = [&](float (&sacc)[2][4], const bool (&valid)[2][2], auto&& vfrag) {
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
    const __half2 p01 = __floats2half2_rn(exp2f(x[0] - mnew), exp2f(x[1] - mnew));
    const __half2 p23 = __floats2half2_rn(exp2f(x[2] - mnew), exp2f(x[3] - mnew));
    const float2 f01 = __half22float2(p01), f23 = __half22float2(p23);
    lrun = lrun * fac + ((f01.x + f01.y) + (f23.x + f23.y));
    const float fa = __shfl_sync(0xffffffffu, fac, 8 * t4);
    const float fb = __shfl_sync(0xffffffffu, fac, 8 * t4 + 4);
#pragma unroll
    for (int m = 0; m < 8; ++m) { o[m][0] *= fa; o[m][1] *= fb; o[m][2] *= fa; o[m][3] *= fb; }
#pragma unroll
    for (int mp = 0; mp < 4; ++mp) {
      uint32_t v[2][4];      // [m - 2mp][a0..a3]
      vfrag(mp, v);
      mma16816(o[2 * mp], v[0][0], v[0][1], v[0][2], v[0][3], h2u(p01), h2u(p23));
      mma16816(o[2 * mp + 1], v[1][0], v[1][1], v[1][2], v[1][3], h2u(p01), h2u(p23));
    }
  };

  // -- forced rows (sinks then recents), pre-packed by pack_forced_kernel as fp16 fragments
  for (int blk = warp; blk < nbf; blk += DW) {
    const int base = blk * 16;
    const uint4* fk = reinterpret_cast<const uint4*>(a.ffrag + ((u * a.fblocks + blk) * 2 * 32 + lane) * 32);
    const uint4* fv = fk + 32 * 8;
    uint32_t kwd[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 t = __ldg(fk + i);
      kwd[4 * i] = t.x; kwd[4 * i + 1] = t.y; kwd[4 * i + 2] = t.z; kwd[4 * i + 3] = t.w;
    }
    uint32_t vwd[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 t = __ldg(fv + i);
      vwd[4 * i] = t.x; vwd[4 * i + 1] = t.y; vwd[4 * i + 2] = t.z; vwd[4 * i + 3] = t.w;
    }
    float sacc[2][4];
    bool valid[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s)
        mma16816(sacc[nt], qa[s][0], 0u, qa[s][1], 0u, kwd[nt * 16 + 2 * s], kwd[nt * 16 + 2 * s + 1]);
      valid[nt][0] = base + 2 * t4 + 8 * nt < nf;
      valid[nt][1] = base + 2 * t4 + 1 + 8 * nt < nf;
    }
    softmax_pv(sacc, valid, [&](int mp, uint32_t (&v)[2][4]) {
#pragma unroll
      for (int mm = 0; mm < 2; ++mm)
#pragma unroll
        for (int r = 0; r < 4; ++r) v[mm][r] = vwd[(2 * mp + mm) * 4 + r];
    });
  }

  PROF(6);
  // -- dynamic rows: cp.async double-buffered staging, dequantised into mma fragments
  const int first = (warp - nbf % DW + DW) % DW;   // this warp's first dynamic block
  if (first < nbd) stage_block(stage, recs, dyn, first * 16, ndyn, lane);
  cp_commit();
  int buf = 0;
  for (int db = first; db < nbd; db += DW) {
    if (db + DW < nbd) stage_block(stage + (buf ^ 1) * STAGE_BYTES, recs, dyn, (db + DW) * 16, ndyn, lane);
    cp_commit();
    cp_wait<1>();
    __syncwarp();
    const char* sb = stage + buf * STAGE_BYTES;
    const int base = db * 16;
    float sacc[2][4];
    bool valid[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int j = g + 8 * nt;
      const uint2 kw = *reinterpret_cast<const uint2*>(chunk(sb, j, t4 >> 1) + 8 * (t4 & 1));
      const uint4 kp = *reinterpret_cast<const uint4*>(chunk(sb, j, 4));
      const uint32_t ks = *reinterpret_cast<const uint32_t*>(chunk(sb, j, 6) + 4 * t4);
      const uint32_t par[4] = {kp.x, kp.y, kp.z, kp.w};
      sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int uu = s >> 2, grp = s >> 1;
        const uint32_t wd = uu ? kw.y : kw.x;
        const __half2 qs2 = u2h(prmt(par[grp], par[grp], 0x1010u));
        const __half2 zp2 = u2h(prmt(par[grp], par[grp], 0x3232u));
        uint32_t b[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = ((s & 3) << 1) | e;
          const uint32_t src = i < 4 ? wd : (wd >> 8);
          const int ii = i & 3;
          const uint32_t xx = lop3_and_or(src, 0x00030003u << (2 * ii), magic[ii]);
          const __half2 c = __hsub2(u2h(xx), u2h(magic[ii]));
          const uint32_t v = h2u(__hfma2(c, qs2, zp2));
          b[e] = lop3_xor_and(v, ks << (15 - (8 * uu + i)), 0x80008000u);
        }
        mma16816(sacc[nt], qa[s][0], 0u, qa[s][1], 0u, b[0], b[1]);
      }
      valid[nt][0] = base + 2 * t4 + 8 * nt < ndyn;
      valid[nt][1] = base + 2 * t4 + 1 + 8 * nt < ndyn;
    }
    // V words and params of tokens 2t4, 2t4+1, 2t4+8, 2t4+9
    uint32_t vw[4];
    uint4 vp[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int j = 2 * t4 + (x & 1) + 8 * (x >> 1);
      vw[x] = *reinterpret_cast<const uint32_t*>(chunk(sb, j, 2 + (g >> 2)) + 4 * (g & 3));
      vp[x] = *reinterpret_cast<const uint4*>(chunk(sb, j, 5));
    }
    softmax_pv(sacc, valid, [&](int jg, uint32_t (&v)[2][4]) {
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const uint32_t pa[4] = {vp[2 * pr].x, vp[2 * pr].y, vp[2 * pr].z, vp[2 * pr].w};
        const uint32_t pb[4] = {vp[2 * pr + 1].x, vp[2 * pr + 1].y, vp[2 * pr + 1].z, vp[2 * pr + 1].w};
        const uint32_t xj = prmt(vw[2 * pr], vw[2 * pr + 1],
                                 (uint32_t)(jg | (jg << 4) | ((4 + jg) << 8) | ((4 + jg) << 12)));
        const __half2 qs2 = u2h(prmt(pa[jg], pb[jg], 0x5410u));
        const __half2 zp2 = u2h(prmt(pa[jg], pb[jg], 0x7632u));
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const uint32_t xx = lop3_and_or(xj, 0x00030003u << (2 * ii), magic[ii]);
          const __half2 c = __hsub2(u2h(xx), u2h(magic[ii]));
          // m = 2jg + (ii >> 1), e = ii & 1 -> a-register 2*pr + e of fragment m
          v[ii >> 1][2 * pr + (ii & 1)] = h2u(__hfma2(c, qs2, zp2));
        }
      }
    });
    __syncwarp();
    buf ^= 1;
  }
  cp_wait<0>();

  PROF(7);
  // ---------------- merge the 8 warp partials (fixed order)
  __syncthreads();
  PROF(8);
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
  PROF(9);
#undef PROF
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
static int align128(int x) { return (x + 127) & ~127; }

DecodeLayout decode_layout(int64_t L, int k, int S, int Gq, int cap) {
  DecodeLayout d{};
  const int W = (int)((L + 31) / 32);
  const int keff = (int)std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  d.capw = std::max(32, cap / DW);
  // R0: pair table while scoring; afterwards hist | gt | eq | dynamic list | staging
  d.off_bits = align128(NBIN * 4);
  d.off_dyn = align128(d.off_bits + 2 * W * 4);
  d.off_stage = align128(d.off_dyn + std::max(keff, 1) * 4);
  const int r0 = std::max(TBL_BYTES, d.off_stage + DW * 2 * STAGE_BYTES);
  // R1: per-warp candidate segments; at other times the tau histogram, the fallback
  // histogram + bitmaps, and the attention partials
  int r1 = DW * d.capw * 8;
  r1 = std::max(r1, NBIN * 4 + 2 * W * 4);
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
                          int fblocks, int R, const float* q, int64_t U, int64_t L, int Gq, int k, int cap,
                          float* out, float* lse, int32_t* sel, int sel_stride, int32_t* sel_count,
                          int32_t* diag, cudaStream_t st, int* smem_out) {
  DecodeLayout d = decode_layout(L, k, S, Gq, cap);
  if (smem_out) *smem_out = d.total;
  DecodeArgs a{signs, recs, cent32, alpha32, sink_idx, ffrag, q, out, lse, sel,
               sel_count, diag, L, fblocks, S, R, Gq, k, d.capw, sel_stride,
               d.off_cand, d.off_forced, d.off_misc, d.off_bits, d.off_dyn, d.off_stage};
  cudaError_t e = cudaFuncSetAttribute(decode_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, d.total);
  if (e != cudaSuccess) return e;
  decode_step_kernel<<<(unsigned)U, DT, d.total, st>>>(a);
  return cudaGetLastError();
}

// Forced rows (sinks then recents) -> fp16 mma fragments, one warp per (unit, 16-row block).
// K^ = K' / alpha-hat (alpha folded into the query), V as is; rows >= S + R are zero.
__global__ void pack_forced_kernel(const float* __restrict__ sink_k, const float* __restrict__ sink_v, int S,
                                   const float* __restrict__ rec_k, const float* __restrict__ rec_v, int64_t rcap,
                                   int R, const float* __restrict__ alpha32, int fblocks, int b0,
                                   uint32_t* __restrict__ frag) {
  const int64_t u = blockIdx.y;
  const int blk = b0 + blockIdx.x, lane = threadIdx.x;
  const int g = lane >> 2, t4 = lane & 3;
  const int nf = S + R;
  auto row = [&](int f, bool key) -> const float* {
    if (f >= nf) return nullptr;
    if (f < S) return (key ? sink_k : sink_v) + (u * S + f) * FD;
    return (key ? rec_k : rec_v) + (u * rcap + (f - S)) * FD;
  };
  auto inva = [&](int d) {
    const float al = alpha32[u * FD + d];
    return 1.0f / (al > 0.f ? al : 1.0f);
  };
  uint32_t* out = frag + ((u * fblocks + blk) * 2 * 32 + lane) * 32;
  const int base = blk * 16;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const float* kr = row(base + g + 8 * nt, true);
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int d = 16 * s + 2 * t4 + 8 * e;
        const float x0 = kr ? kr[d] * inva(d) : 0.f, x1 = kr ? kr[d + 1] * inva(d + 1) : 0.f;
        out[nt * 16 + 2 * s + e] = h2u(__floats2half2_rn(x0, x1));
      }
  }
  uint32_t* ov = out + 32 * 32;
#pragma unroll
  for (int m = 0; m < 8; ++m)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int d = 16 * m + g + 8 * (r & 1), pr = r >> 1;
      const float* va = row(base + 2 * t4 + 8 * pr, false);
      const float* vb = row(base + 2 * t4 + 8 * pr + 1, false);
      ov[m * 4 + r] = h2u(__floats2half2_rn(va ? va[d] : 0.f, vb ? vb[d] : 0.f));
    }
}

cudaError_t launch_pack_forced(const float* sink_k, const float* sink_v, int S, const float* rec_k,
                               const float* rec_v, int64_t rcap, int R, const float* alpha32, int64_t U,
                               int fblocks, int b0, int b1, uint32_t* frag, cudaStream_t st) {
  if (b1 <= b0 || U == 0) return cudaSuccess;
  pack_forced_kernel<<<dim3(b1 - b0, (unsigned)U), 32, 0, st>>>(sink_k, sink_v, S, rec_k, rec_v, rcap, R,
                                                               alpha32, fblocks, b0, frag);
  return cudaGetLastError();
}

cudaError_t set_decode_profile(long long* p) {
  return cudaMemcpyToSymbol(g_prof, &p, sizeof(p));
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
