// Device building blocks of the fused decode step, shared by the one-unit-per-CTA kernel
// (decode.cu), the cluster-split kernel (decode_split.cu) and the two-kernel path (decode_two.cu).
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace sikv {

constexpr int TBL_BYTES = 256 * 64 * 4;   // pair table: 256 byte values x 64 columns
constexpr int NB = 8;                     // chunks (of 256 tokens) scored per thread per batch
constexpr int STAGE_BYTES = 16 * FREC;    // one 16-token block of records
constexpr int MAX_SAMPLE_CHUNKS = 8;
// sample chunks are at least SSTRIDE_MIN chunks apart (>= NB: one per B2 batch at most), so
// short units (< 32K tokens) still sample up to 8 chunks: a tighter threshold, fewer candidates
constexpr int SSTRIDE_MIN = 8;
static_assert(SSTRIDE_MIN >= NB, "at most one sample chunk per B2 batch (the stride is rounded to a multiple of NB)");

// ---------------------------------------------------------------- pair table
// LUT[g][c] = q-bar_g . centroid[g][c] (float32, no FMA, the reference pairing) and the
// byte-pair table T[b][col] = LUT[2p][b & 15] + LUT[2p+1][b >> 4], p = col mod 16.
// T rows from the transposed LUT lutT[code * 32 + group]: lanes 0-15 / 16-31 build pairs
// p = lane & 15 of two byte values, so LUT reads hit banks 2p, 2p+1 and T writes banks p.
template <class Grp>
__device__ __forceinline__ void build_pair_rows(const float* lutT, char* T) {
  const int tid = Grp::tid();
  const int p = tid & 15;
  for (int b = tid >> 4; b < 256; b += DT / 16) {
    const float v = __fadd_rn(lutT[(b & 15) * 32 + 2 * p], lutT[(b >> 4) * 32 + 2 * p + 1]);
    float* row = reinterpret_cast<float*>(T) + b * 64;
    row[p] = v; row[p + 16] = v; row[p + 32] = v;
  }
  Grp::sync();
}

// 32-column variant (ColKey): T[b][16 h + p] (two copies, row stride 256 B; the caller
// offsets T by 128 B for the second buffer).  Lanes 16-31 write the other copy first, so
// both stores of a warp hit 32 distinct banks.
template <class Grp>
__device__ __forceinline__ void build_pair_rows_col(const float* lutT, char* T) {
  const int tid = Grp::tid();
  const int p = tid & 15, hh = (tid >> 4) & 1;
  for (int b = tid >> 4; b < 256; b += DT / 16) {
    const float v = __fadd_rn(lutT[(b & 15) * 32 + 2 * p], lutT[(b >> 4) * 32 + 2 * p + 1]);
    float* row = reinterpret_cast<float*>(T) + b * 64;
    row[p + 16 * hh] = v;
    row[p + 16 * (1 - hh)] = v;
  }
  Grp::sync();
}

// The four factors of LUT entry (group g, code c): its centroid, or for the sign-only ablation
// (build_sign_lut, retrieval.py:54-62) the code's +-1 pattern (element i <-> bit 3 - i); the
// products with q-bar are then exact and the stated pairing is unchanged.
__device__ __forceinline__ float4 lut_factors(float4 c, int code, int sign_only) {
  if (!sign_only) return c;
  return make_float4((code & 8) ? 1.f : -1.f, (code & 4) ? 1.f : -1.f, (code & 2) ? 1.f : -1.f,
                     (code & 1) ? 1.f : -1.f);
}

template <class Grp>
__device__ __forceinline__ void build_pair_table(const float* __restrict__ cent, const float* qbar, float* lut,
                                                 char* T, int sign_only = 0) {
  const int tid = Grp::tid();
  for (int e = tid; e < 512; e += DT) {
    const int g = e >> 4;
    const float4 c = lut_factors(reinterpret_cast<const float4*>(cent)[e], e & 15, sign_only);
    const float q0 = qbar[4 * g], q1 = qbar[4 * g + 1], q2 = qbar[4 * g + 2], q3 = qbar[4 * g + 3];
    lut[(e & 15) * 32 + g] = __fadd_rn(__fadd_rn(__fmul_rn(q0, c.x), __fmul_rn(q2, c.z)),
                                       __fadd_rn(__fmul_rn(q1, c.y), __fmul_rn(q3, c.w)));
  }
  Grp::sync();
  build_pair_rows<Grp>(lut, T);
}

// ---------------------------------------------------------------- scoring
// A lane's table addressing.  RepKey: the 64-column table of build_pair_rows (pair p
// replicated at columns p, p+16, p+32), the lane's column at step i is lb + i (folded into
// the LDS immediate).  ColKey: the 32-column table of build_pair_rows_col (two copies of the
// 16 pairs, one per half warp); a row stride of 256 B leaves room for a second buffer, so
// two tables interleave in one 64 KiB region.  The lane's 16 column offsets (pair (j+i) mod
// 16 of its half-warp copy) sit in 4 registers and the PRMT that extracts the sign byte also
// picks the column byte (sign-replicating selectors zero the high bytes: offsets < 128).
// Both are bank-conflict free: the 32 lanes of a step hit 32 distinct columns mod 32.
struct RepKey {
  uint32_t lb;
  __device__ __forceinline__ explicit RepKey(int lane) : lb((uint32_t)(64 * ((lane >> 4) & 1) + 4 * (lane & 15))) {
    asm volatile("" : "+r"(lb));     // kept in a register (not rematerialised per batch)
  }
  __device__ __forceinline__ uint32_t off(uint32_t w, int i) const {
    return prmt(w, lb, 0x5504u | ((uint32_t)(i & 3) << 4)) + 4 * i;
  }
};
struct ColKey {
  uint32_t c[4];
  __device__ __forceinline__ explicit ColKey(int lane) {
    const int h = (lane >> 4) & 1, j = lane & 15;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = 0;
#pragma unroll
      for (int m = 0; m < 4; ++m) v |= (uint32_t)(4 * (16 * h + ((j + 4 * k + m) & 15))) << (8 * m);
      c[k] = v;
      // opaque to the compiler: kept in registers instead of being rematerialised from the
      // lane id inside every scoring batch (~25 integer instructions per batch)
      asm volatile("" : "+r"(c[k]));
    }
  }
  __device__ __forceinline__ uint32_t off(uint32_t w, int i) const {
    const uint32_t m = (uint32_t)(i & 3);
    return prmt(w, c[i >> 2], (4u + m) | (m << 4) | ((12u + m) << 8) | ((12u + m) << 12));
  }
};

// score of the token whose 16-byte rotated sign record is w; T = pair table (row stride
// 256 B).  Pairs are summed left to right starting at pair (t mod 16) — the order
// oracle/restate32.py states.
template <class Key>
__device__ __forceinline__ float score_token(const uint4 w, const Key& key, const char* T) {
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float v = *reinterpret_cast<const float*>(T + key.off(ww[i >> 2], i));
    s = (i == 0) ? v : __fadd_rn(s, v);
  }
  return s;
}

// N tokens at once: the 16-step chains of different tokens interleave, hiding FADD latency.
// Pairs of tokens accumulate with one packed FADD2 (add.rn.f32x2, sm_100a): per lane it is
// the same correctly rounded float32 add, so the stated order and the bits are unchanged.
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

template <int N, class Key>
__device__ __forceinline__ void score_batch(const uint4 (&w)[N], const Key& key, const char* T, float (&s)[N]) {
  static_assert(N % 2 == 0, "tokens are scored in pairs");
  unsigned long long acc[N / 2];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int x = 0; x < N; x += 2) {
      const uint32_t w0 = (i >> 2) == 0 ? w[x].x : (i >> 2) == 1 ? w[x].y : (i >> 2) == 2 ? w[x].z : w[x].w;
      const uint32_t w1 = (i >> 2) == 0 ? w[x + 1].x : (i >> 2) == 1 ? w[x + 1].y : (i >> 2) == 2 ? w[x + 1].z
                                                                                               : w[x + 1].w;
      const float v0 = *reinterpret_cast<const float*>(T + key.off(w0, i));
      const float v1 = *reinterpret_cast<const float*>(T + key.off(w1, i));
      const unsigned long long v = pack2(v0, v1);
      acc[x / 2] = (i == 0) ? v : fadd2(acc[x / 2], v);
    }
  }
#pragma unroll
  for (int x = 0; x < N; x += 2) unpack2(acc[x / 2], s[x], s[x + 1]);
}

// streaming 16-byte load of the sign plane: read once, no L1 allocation, and first out of L2
// (the dynamic lists and queries the attention reads next stay resident instead)
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ bool forced_bit(const uint32_t* fb, int64_t t) {
  return (fb[t >> 5] >> (t & 31)) & 1u;
}

__device__ __forceinline__ uint32_t unkey_bits(uint32_t k2) {
  return (k2 & 0x80000000u) ? (k2 & 0x7FFFFFFFu) : ~k2;
}

// f32_key in three instructions: x + 0 turns -0 into +0 (round-to-nearest), then the sign
// mask flips the negatives and sets the top bit of the positives
__device__ __forceinline__ uint32_t f32_key_fast(float x) {
  const uint32_t u = __float_as_uint(__fadd_rn(x, 0.0f));
  return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}

// v[x] for a run-time x in [0, N): a select tree on the bits of x (N = 4 or 8)
template <int N>
__device__ __forceinline__ float pick_dyn(const float (&v)[N], int x) {
  static_assert(N == 4 || N == 8, "pick_dyn supports 4 or 8 values");
  const bool b0 = x & 1, b1 = x & 2;
  const float a01 = b0 ? v[1] : v[0], a23 = b0 ? v[3] : v[2];
  const float lo = b1 ? a23 : a01;
  if constexpr (N == 4) {
    return lo;
  } else {
    const float a45 = b0 ? v[5] : v[4], a67 = b0 ? v[7] : v[6];
    const float hi = b1 ? a67 : a45;
    return (x & 4) ? hi : lo;
  }
}

// predicated 8-byte shared-memory store (no branch)
__device__ __forceinline__ void st_shared_v2_if(bool p, uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.u32 [%1], {%2, %3}; }"
               ::"r"((uint32_t)p), "r"(addr), "r"(a), "r"(b));
}

// ---------------------------------------------------------------- async staging
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// staged-record swizzle: 16-byte chunk kk of block token j lives at slot kk ^ stage_sw(j).
// Conflict-free for the fragment reads below: K4 chunks t4 of tokens 2p, 2p+1 fill all 8
// slots of a quarter-warp phase; the V words / params of the 4 even (odd) tokens of a block
// hit 4 distinct slot pairs.
__host__ __device__ __forceinline__ int stage_sw(int j) { return (j & 6) ^ ((j & 1) << 2); }

// two e2m1 nibbles (byte B of w) -> f16x2 (lo nibble -> low half)
template <int B>
__device__ __forceinline__ uint32_t e2m1x2_to_h2(uint32_t w) {
  uint32_t r;
  if constexpr (B == 0)
    asm("{ .reg .b8 b0, b1, b2, b3; mov.b32 {b0, b1, b2, b3}, %1; cvt.rn.f16x2.e2m1x2 %0, b0; }" : "=r"(r) : "r"(w));
  else if constexpr (B == 1)
    asm("{ .reg .b8 b0, b1, b2, b3; mov.b32 {b0, b1, b2, b3}, %1; cvt.rn.f16x2.e2m1x2 %0, b1; }" : "=r"(r) : "r"(w));
  else if constexpr (B == 2)
    asm("{ .reg .b8 b0, b1, b2, b3; mov.b32 {b0, b1, b2, b3}, %1; cvt.rn.f16x2.e2m1x2 %0, b2; }" : "=r"(r) : "r"(w));
  else
    asm("{ .reg .b8 b0, b1, b2, b3; mov.b32 {b0, b1, b2, b3}, %1; cvt.rn.f16x2.e2m1x2 %0, b3; }" : "=r"(r) : "r"(w));
  return r;
}

// K^ for two channels from their e2m1 byte: (2 qs) x + copysign(zp, x), x = sign * code / 2.
// Bit-identical to sign * fl16(qs c + zp) (c/2 * 2qs is exact; one rounding, symmetric).
template <int B>
__device__ __forceinline__ uint32_t k_dequant2(uint32_t w, __half2 qs2, uint32_t zp2) {
  const uint32_t x = e2m1x2_to_h2<B>(w);
  uint32_t z;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(z) : "r"(x), "r"(0x80008000u), "r"(zp2));   // (x & m) | zp
  return h2u(__hfma2(u2h(x), qs2, u2h(z)));
}

// ---------------------------------------------------------------- sparse attention
// One warp's flash-decode state for the unit's GQA group.  QK^T runs as S^T = K^ q~^T (M = 16
// tokens of a block, N = 8 heads, K = channels): q~ is the B operand (qa[s] = b0, b1 of k-step
// s: head g, channels 16 s + 2 t4 (+ 8)) and a thread's scores are (tokens g, g + 8) x (heads
// 2 t4, 2 t4 + 1).  PV runs as O^T = V^T P (M = 128 channels as 8 m-tiles, N = 8 heads), so a
// thread's O accumulators belong to the same two heads: mrun / lrun per head h0 = 2 t4,
// h1 = 2 t4 + 1 (lrun: this thread's tokens only, summed over the g lanes at the end).
struct Attn {
  uint32_t qa[8][2];
  float o[8][4];
  float mrun[2], lrun[2];
};

// log2(e) / sqrt(128): folded into q~, so the MMA yields the exp2-domain logits directly
constexpr float kSoftmaxScale = 1.4426950408889634f * 0.08838834764831845f;

// q~ = q * alpha-hat * kSoftmaxScale straight from global memory (each warp on its own)
__device__ __forceinline__ void attn_init_g(Attn& A, const float* __restrict__ q_u, const float* __restrict__ alpha_u,
                                            int Gq, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  const int gg = g < Gq ? g : 0;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int d = 16 * s + 2 * t4 + 8 * e;
      const float2 qv = __ldg(reinterpret_cast<const float2*>(q_u + gg * FD + d));
      const float2 av = __ldg(reinterpret_cast<const float2*>(alpha_u + d));
      const float a0 = av.x > 0.f ? av.x : 1.0f, a1 = av.y > 0.f ? av.y : 1.0f;
      const float x0 = g < Gq ? qv.x * a0 * kSoftmaxScale : 0.f, x1 = g < Gq ? qv.y * a1 * kSoftmaxScale : 0.f;
      A.qa[s][e] = h2u(__floats2half2_rn(x0, x1));
    }
#pragma unroll
  for (int m = 0; m < 8; ++m) A.o[m][0] = A.o[m][1] = A.o[m][2] = A.o[m][3] = 0.f;
  A.mrun[0] = A.mrun[1] = -INFINITY;
  A.lrun[0] = A.lrun[1] = 0.f;
}

__device__ __forceinline__ void attn_init(Attn& A, const float* qs, const float* ahat, int Gq, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int d = 16 * s + 2 * t4 + 8 * e;
      float x0 = 0.f, x1 = 0.f;
      if (g < Gq) {
        x0 = qs[g * FD + d] * ahat[d] * kSoftmaxScale;
        x1 = qs[g * FD + d + 1] * ahat[d + 1] * kSoftmaxScale;
      }
      A.qa[s][e] = h2u(__floats2half2_rn(x0, x1));
    }
#pragma unroll
  for (int m = 0; m < 8; ++m) A.o[m][0] = A.o[m][1] = A.o[m][2] = A.o[m][3] = 0.f;
  A.mrun[0] = A.mrun[1] = -INFINITY;
  A.lrun[0] = A.lrun[1] = 0.f;
}

constexpr float kLazyRescale = 8.0f;
// 2^x on the SFU (x <= 8 here: logits minus the reference max; -inf -> +0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fp16 magic for a 2-bit code at bits [2i, 2i+2) of each half: 2^(10-2i), so that
// (w & mask_i) | magic_i is the half 2^(10-2i) + code exactly
__host__ __device__ constexpr uint32_t kMagic(int i) { return ((25u - 2u * (uint32_t)i) << 10) * 0x00010001u; }

// online softmax update + P V for one 16-token block: sacc = S^T fragment (tokens g, g + 8 x
// heads 2 t4, 2 t4 + 1); rows at block offsets >= rem are padding
template <typename VFrag>
__device__ __forceinline__ void attn_softmax_pv(Attn& A, const float (&sacc)[4], int rem, int lane,
                                                VFrag&& vfrag) {
  const int g = lane >> 2;
  float x[4];
  x[0] = g < rem ? sacc[0] : -INFINITY;       // token g, head h0 (exp2-domain logits: q~ is prescaled)
  x[1] = g < rem ? sacc[1] : -INFINITY;       // token g, head h1
  x[2] = g + 8 < rem ? sacc[2] : -INFINITY;   // token g + 8, head h0
  x[3] = g + 8 < rem ? sacc[3] : -INFINITY;   // token g + 8, head h1
  // lazy rescale: the reference max only moves when the block max exceeds it by more than
  // 2^8 (exp2 domain), so P <= 256 (exact range in fp16) and most blocks skip the O rescale.
  // The block max is only reduced when some score exceeds the bound (the same decision as
  // comparing the reduced block max, without its shuffles in the common case).
  const float lim0 = A.mrun[0] + kLazyRescale, lim1 = A.mrun[1] + kLazyRescale;
  if (__any_sync(0xffffffffu, x[0] > lim0 || x[2] > lim0 || x[1] > lim1 || x[3] > lim1)) {
    float bm0 = fmaxf(x[0], x[2]), bm1 = fmaxf(x[1], x[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
    }
    const float mn0 = bm0 > lim0 ? bm0 : A.mrun[0];
    const float mn1 = bm1 > lim1 ? bm1 : A.mrun[1];
    const float fa = ex2(A.mrun[0] - mn0), fb = ex2(A.mrun[1] - mn1);
    A.mrun[0] = mn0;
    A.mrun[1] = mn1;
    A.lrun[0] *= fa;
    A.lrun[1] *= fb;
#pragma unroll
    for (int m = 0; m < 8; ++m) { A.o[m][0] *= fa; A.o[m][1] *= fb; A.o[m][2] *= fa; A.o[m][3] *= fb; }
  }
  const float mn0 = A.mrun[0], mn1 = A.mrun[1];
  const __half2 p0 = __floats2half2_rn(ex2(x[0] - mn0), ex2(x[1] - mn1));   // token g: heads h0, h1
  const __half2 p1 = __floats2half2_rn(ex2(x[2] - mn0), ex2(x[3] - mn1));   // token g + 8
  const float2 f0 = __half22float2(p0), f1 = __half22float2(p1);
  A.lrun[0] += f0.x + f1.x;
  A.lrun[1] += f0.y + f1.y;
  // P as the PV B operand (tokens 2 t4, 2 t4 + 1 (+ 8) x head g): one transpose per 8 tokens
  const uint32_t pb0 = movmatrix_trans(h2u(p0)), pb1 = movmatrix_trans(h2u(p1));
#pragma unroll
  for (int mp = 0; mp < 4; ++mp) {
    uint32_t v[2][4];      // [m - 2mp][a0..a3]
    vfrag(mp, v);
    mma16816(A.o[2 * mp], v[0][0], v[0][1], v[0][2], v[0][3], pb0, pb1);
    mma16816(A.o[2 * mp + 1], v[1][0], v[1][1], v[1][2], v[1][3], pb0, pb1);
  }
}

// forced rows (sinks then recents), pre-packed as fp16 fragments with per-row scales
// (FBLK_WORDS per 16-row block); this warp takes blocks wi, wi + nw, ... of [0, nbf)
__device__ __forceinline__ void attn_forced(Attn& A, const uint32_t* ffrag_u, int nf, int wi, int nw, int lane) {
  const int nbf = (nf + 15) >> 4;
  const int g = lane >> 2;
  for (int blk = wi; blk < nbf; blk += nw) {
    const int base = blk * 16;
    const uint32_t* fb = ffrag_u + (int64_t)blk * FBLK_WORDS;
    const uint4* fk = reinterpret_cast<const uint4*>(fb + lane * 32);
    const uint4* fv = fk + 32 * 8;
    const float sc0 = __ldg(reinterpret_cast<const float*>(fb + 2 * 32 * 32) + g);       // row g
    const float sc1 = __ldg(reinterpret_cast<const float*>(fb + 2 * 32 * 32) + 8 + g);   // row g + 8
    uint32_t kwd[32], vwd[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 t = __ldg(fk + i);
      kwd[4 * i] = t.x; kwd[4 * i + 1] = t.y; kwd[4 * i + 2] = t.z; kwd[4 * i + 3] = t.w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 t = __ldg(fv + i);
      vwd[4 * i] = t.x; vwd[4 * i + 1] = t.y; vwd[4 * i + 2] = t.z; vwd[4 * i + 3] = t.w;
    }
    float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < 8; ++s)
      mma16816(sacc, kwd[2 * s], kwd[16 + 2 * s], kwd[2 * s + 1], kwd[16 + 2 * s + 1], A.qa[s][0], A.qa[s][1]);
    sacc[0] *= sc0; sacc[1] *= sc0; sacc[2] *= sc1; sacc[3] *= sc1;
    attn_softmax_pv(A, sacc, nf - base, lane, [&](int mp, uint32_t (&v)[2][4]) {
#pragma unroll
      for (int mm = 0; mm < 2; ++mm)
#pragma unroll
        for (int r = 0; r < 4; ++r) v[mm][r] = vwd[(2 * mp + mm) * 4 + r];
    });
  }
}

// fragment offsets of a lane inside a staged 16-token block (token g for K, tokens 2t4 /
// 2t4 + 1 for V; the +8 tokens are P8 bytes further)
struct BlkOffs {
  int k4, kp, vw0, vw1, vp0, vp1;
};
constexpr int P8 = 8 * FREC;

// QK^T, online softmax and PV of one staged 16-token block (rem = valid rows from its start)
__device__ __forceinline__ void attn_block(Attn& A, const char* sb, const BlkOffs& o, int rem, int lane) {
  float sacc[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t kw[2][4], par[2][4];     // tokens g, g + 8
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const uint4 k4 = *reinterpret_cast<const uint4*>(sb + o.k4 + nt * P8);
    const uint4 kp = *reinterpret_cast<const uint4*>(sb + o.kp + nt * P8);
    kw[nt][0] = k4.x; kw[nt][1] = k4.y; kw[nt][2] = k4.z; kw[nt][3] = k4.w;
    par[nt][0] = kp.x; par[nt][1] = kp.y; par[nt][2] = kp.z; par[nt][3] = kp.w;
  }
#pragma unroll
  for (int grp = 0; grp < 4; ++grp) {
    const __half2 qa2 = __low2half2(u2h(par[0][grp])), qb2 = __low2half2(u2h(par[1][grp]));   // HFMA2 .H0_H0 operands
    const uint32_t za2 = prmt(par[0][grp], par[0][grp], 0x3232u), zb2 = prmt(par[1][grp], par[1][grp], 0x3232u);
    // k-steps s = 2 grp (bytes 0, 1 of word grp) and 2 grp + 1 (bytes 2, 3); A rows g / g + 8
    mma16816(sacc, k_dequant2<0>(kw[0][grp], qa2, za2), k_dequant2<0>(kw[1][grp], qb2, zb2),
             k_dequant2<1>(kw[0][grp], qa2, za2), k_dequant2<1>(kw[1][grp], qb2, zb2), A.qa[2 * grp][0],
             A.qa[2 * grp][1]);
    mma16816(sacc, k_dequant2<2>(kw[0][grp], qa2, za2), k_dequant2<2>(kw[1][grp], qb2, zb2),
             k_dequant2<3>(kw[0][grp], qa2, za2), k_dequant2<3>(kw[1][grp], qb2, zb2), A.qa[2 * grp + 1][0],
             A.qa[2 * grp + 1][1]);
  }
  // V words and params of tokens 2t4, 2t4+1, 2t4+8, 2t4+9
  uint32_t vw[4];
  uint4 vp[4];
  vw[0] = *reinterpret_cast<const uint32_t*>(sb + o.vw0);
  vw[1] = *reinterpret_cast<const uint32_t*>(sb + o.vw1);
  vw[2] = *reinterpret_cast<const uint32_t*>(sb + o.vw0 + P8);
  vw[3] = *reinterpret_cast<const uint32_t*>(sb + o.vw1 + P8);
  vp[0] = *reinterpret_cast<const uint4*>(sb + o.vp0);
  vp[1] = *reinterpret_cast<const uint4*>(sb + o.vp1);
  vp[2] = *reinterpret_cast<const uint4*>(sb + o.vp0 + P8);
  vp[3] = *reinterpret_cast<const uint4*>(sb + o.vp1 + P8);
  attn_softmax_pv(A, sacc, rem, lane, [&](int jg, uint32_t (&v)[2][4]) {
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
        const uint32_t xx = lop3_and_or(xj, 0x00030003u << (2 * ii), kMagic(ii));
        const __half2 c = __hsub2(u2h(xx), u2h(kMagic(ii)));
        // m = 2jg + (ii >> 1), e = ii & 1 -> a-register 2*pr + e of fragment m
        v[ii >> 1][2 * pr + (ii & 1)] = h2u(__hfma2(c, qs2, zp2));
      }
    }
  });
}

// dynamic rows: blocks first, first + nw, ... of [0, nbd), staged by cp.async (NSTAGE
// buffers per warp: NSTAGE - 1 blocks in flight) and dequantised into mma fragments.  The list is padded to a multiple of 16
// (pad_dyn), so staging needs no bounds.  Every lane's shared-memory offsets are fixed for
// the whole unit (16-byte chunk k of token j lives at chunk k ^ (j & 7)), so they are
// computed once; token g and g + 8 (and 2t4 + x and 2t4 + x + 8) differ by 1 KiB.
struct NoPrologue {
  __device__ __forceinline__ void operator()() const {}
};
// `pro` runs once the first blocks' gathers are in flight (e.g. the q~ setup and the forced
// rows, so their latencies overlap those of the list and the gathers)
template <int NSTAGE = 2, class Pro = NoPrologue>
__device__ __forceinline__ void attn_dynamic(Attn& A, const uint8_t* recs_u, const int32_t* dyn, int ndyn,
                                             int first, int nw, char* stage, int lane, Pro pro = Pro()) {
  const int g = lane >> 2, t4 = lane & 3;
  const int nbd = (ndyn + 15) >> 4;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage);
  // staging: lane copies chunk kk = lane & 7 of tokens j = 4 (lane >> 3) + r, r = 0..3 (its
  // four row indices are one 16-byte load of the list)
  const int jb = lane >> 3, kk = lane & 7;
  uint32_t dst[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int j = 4 * jb + r;
    dst[r] = (uint32_t)(j * FREC + 16 * (kk ^ stage_sw(j)));
  }
  const uint8_t* src0 = recs_u + 16 * kk;
  // the row indices of the block staged next are loaded one block ahead (registers), so the
  // list read (shared or global memory) is off the staging path
  int32_t tix[4];
  auto load_ix = [&](int blk) {
    const int4 v = *reinterpret_cast<const int4*>(dyn + blk * 16 + 4 * jb);
    tix[0] = v.x; tix[1] = v.y; tix[2] = v.z; tix[3] = v.w;
  };
  auto stage_blk = [&](uint32_t buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint8_t* src = src0 + (size_t)((uint32_t)tix[r] * (uint32_t)FREC);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + buf + dst[r]), "l"(src));
    }
  };
  // fragment offsets (token g for K, tokens 2t4 / 2t4 + 1 for V; +1 KiB for the +8 tokens)
  const int jk = g, jv0 = 2 * t4, jv1 = 2 * t4 + 1;
  BlkOffs o;
  o.k4 = jk * FREC + 16 * (t4 ^ stage_sw(jk));
  o.kp = jk * FREC + 16 * (6 ^ stage_sw(jk));
  o.vw0 = jv0 * FREC + 16 * ((4 + (g >> 2)) ^ stage_sw(jv0)) + 4 * (g & 3);
  o.vw1 = jv1 * FREC + 16 * ((4 + (g >> 2)) ^ stage_sw(jv1)) + 4 * (g & 3);
  o.vp0 = jv0 * FREC + 16 * (7 ^ stage_sw(jv0));
  o.vp1 = jv1 * FREC + 16 * (7 ^ stage_sw(jv1));
  // prologue: the next block's indices are requested before this block's wait on its own
  if (first < nbd) load_ix(first);
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    const int bn = first + (s + 1) * nw;
    int32_t tn[4] = {0, 0, 0, 0};
    if (bn < nbd) {
      const int4 v = *reinterpret_cast<const int4*>(dyn + bn * 16 + 4 * jb);
      tn[0] = v.x; tn[1] = v.y; tn[2] = v.z; tn[3] = v.w;
    }
    if (first + s * nw < nbd) stage_blk(s * STAGE_BYTES);
    cp_commit();
#pragma unroll
    for (int r = 0; r < 4; ++r) tix[r] = tn[r];
  }
  pro();
  int buf = 0;
  for (int db = first; db < nbd; db += nw) {
    const int nx = db + (NSTAGE - 1) * nw;
    if (nx < nbd) {
      stage_blk(((buf + NSTAGE - 1) % NSTAGE) * STAGE_BYTES);
      if (nx + nw < nbd) load_ix(nx + nw);
    }
    cp_commit();
    cp_wait<NSTAGE - 1>();
    __syncwarp();
    attn_block(A, stage + buf * STAGE_BYTES, o, ndyn - db * 16, lane);
    __syncwarp();
    buf = buf + 1 == NSTAGE ? 0 : buf + 1;
  }
  cp_wait<0>();
}

// ---- 16-bit records (FREC16): the fragments are stored, no dequantisation
constexpr int STAGE16_BYTES = 16 * FREC16;     // one 16-token block

// QK^T, online softmax and PV of one staged 16-bit block (rem = valid rows from its start)
__device__ __forceinline__ void attn_block16(Attn& A, uint32_t sb, int rem, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {      // k-steps 2i, 2i + 1
    uint32_t kw[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int j = g + 8 * nt;
      uint4 t;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                   : "r"(sb + (uint32_t)(j * FREC16 + 16 * sw16(j, 4 * t4 + i))));
      kw[nt][0] = t.x; kw[nt][1] = t.y; kw[nt][2] = t.z; kw[nt][3] = t.w;
    }
    mma16816(sacc, kw[0][0], kw[1][0], kw[0][1], kw[1][1], A.qa[2 * i][0], A.qa[2 * i][1]);
    mma16816(sacc, kw[0][2], kw[1][2], kw[0][3], kw[1][3], A.qa[2 * i + 1][0], A.qa[2 * i + 1][1]);
  }
  // V words of tokens 2t4, 2t4 + 1, 2t4 + 8, 2t4 + 9: word m of chunk g = (ch 16m + g, 16m + g + 8)
  uint32_t vw[4][8];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int j = 2 * t4 + (x & 1) + 8 * (x >> 1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint4 t;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                   : "r"(sb + (uint32_t)(j * FREC16 + 16 * sw16(j, 16 + 2 * g + h))));
      vw[x][4 * h] = t.x; vw[x][4 * h + 1] = t.y; vw[x][4 * h + 2] = t.z; vw[x][4 * h + 3] = t.w;
    }
  }
  attn_softmax_pv(A, sacc, rem, lane, [&](int mp, uint32_t (&v)[2][4]) {
#pragma unroll
    for (int mm = 0; mm < 2; ++mm) {
      const int m = 2 * mp + mm;
      v[mm][0] = prmt(vw[0][m], vw[1][m], 0x5410u);
      v[mm][1] = prmt(vw[0][m], vw[1][m], 0x7632u);
      v[mm][2] = prmt(vw[2][m], vw[3][m], 0x5410u);
      v[mm][3] = prmt(vw[2][m], vw[3][m], 0x7632u);
    }
  });
}

// dynamic rows from 16-bit records: blocks first, first + nw, ... of [0, nbd), staged by
// cp.async (NSTAGE buffers per warp); lane copies half (16 units) of block token lane >> 1
template <int NSTAGE = 2>
__device__ __forceinline__ void attn_dynamic16(Attn& A, const uint8_t* recs_u, const int32_t* dyn, int ndyn,
                                               int first, int nw, char* stage, int lane) {
  const int nbd = (ndyn + 15) >> 4;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage);
  const int jt = lane >> 1, half = lane & 1;
  int32_t tix = 0;
  auto stage_blk = [&](uint32_t buf) {
    const uint8_t* src = recs_u + (size_t)((uint32_t)tix * (uint32_t)FREC16) + 256 * half;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int u = 16 * half + i;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + buf + (uint32_t)(jt * FREC16 + 16 * sw16(jt, u))),
                   "l"(src + 16 * i));
    }
  };
  if (first < nbd) tix = dyn[first * 16 + jt];
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    const int bn = first + (s + 1) * nw;
    const int32_t tn = bn < nbd ? dyn[bn * 16 + jt] : 0;
    if (first + s * nw < nbd) stage_blk(s * STAGE16_BYTES);
    cp_commit();
    tix = tn;
  }
  int buf = 0;
  for (int db = first; db < nbd; db += nw) {
    const int nx = db + (NSTAGE - 1) * nw;
    if (nx < nbd) {
      stage_blk(((buf + NSTAGE - 1) % NSTAGE) * STAGE16_BYTES);
      if (nx + nw < nbd) tix = dyn[(nx + nw) * 16 + jt];
    }
    cp_commit();
    cp_wait<NSTAGE - 1>();
    __syncwarp();
    attn_block16(A, sbase + buf * STAGE16_BYTES, ndyn - db * 16, lane);
    __syncwarp();
    buf = buf + 1 == NSTAGE ? 0 : buf + 1;
  }
  cp_wait<0>();
}

// this warp's partial (O, m, l) -> shared memory [nw][Gq][128], [nw][Gq], [nw][Gq]
__device__ __forceinline__ void attn_write_partial(const Attn& A, float* part, float* pm, float* pl, int wi,
                                                   int Gq, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  float l0 = A.lrun[0], l1 = A.lrun[1];
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  if (g == 0) {
    if (2 * t4 < Gq) { pm[wi * Gq + 2 * t4] = A.mrun[0]; pl[wi * Gq + 2 * t4] = l0; }
    if (2 * t4 + 1 < Gq) { pm[wi * Gq + 2 * t4 + 1] = A.mrun[1]; pl[wi * Gq + 2 * t4 + 1] = l1; }
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int h0 = 2 * t4, h1 = 2 * t4 + 1, d0 = 16 * m + g, d1 = d0 + 8;
    if (h0 < Gq) { part[(wi * Gq + h0) * FD + d0] = A.o[m][0]; part[(wi * Gq + h0) * FD + d1] = A.o[m][2]; }
    if (h1 < Gq) { part[(wi * Gq + h1) * FD + d0] = A.o[m][1]; part[(wi * Gq + h1) * FD + d1] = A.o[m][3]; }
  }
}

// fixed-order merge of the nw partials (caller synchronises before).  The per-(warp, head)
// factors 2^(m_w - M) replace pm in place and the denominators replace pl[h] (one Grp sync).
template <class Grp>
__device__ __forceinline__ void attn_merge(const float* part, float* pm, float* pl, int nw, int Gq, int gtid,
                                           int gsize, float* out_u, float* lse_u) {
  if (gtid < Gq) {
    const int h = gtid;
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, pm[w * Gq + h]);
    float den = 0.f;
    for (int w = 0; w < nw; ++w) {
      const float mw = pm[w * Gq + h];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      den += pl[w * Gq + h] * f;
      pm[w * Gq + h] = f;
    }
    pl[h] = den;
    if (lse_u) lse_u[h] = (M + log2f(den)) * 0.6931471805599453f;
  }
  Grp::sync();
  // four channels per thread (same per-element order: num += part * factor over w)
  for (int e = gtid; e < Gq * FD / 4; e += gsize) {
    const int h = e / (FD / 4), d4 = e % (FD / 4);
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < nw; ++w) {
      const float4 p = reinterpret_cast<const float4*>(part + (w * Gq + h) * FD)[d4];
      const float f = pm[w * Gq + h];
      num.x += p.x * f; num.y += p.y * f; num.z += p.z * f; num.w += p.w * f;
    }
    const float den = pl[h];
    reinterpret_cast<float4*>(out_u + h * FD)[d4] = make_float4(num.x / den, num.y / den, num.z / den, num.w / den);
  }
}

// merge of the nw warp partials into one CTA partial (caller synchronises before): per head
// num[128] = sum_w part_w 2^(m_w - M), then M, den = sum_w l_w 2^(m_w - M) -> dst[h][FD + 2]
__device__ __forceinline__ void attn_merge_partial(const float* part, float* pm, const float* pl, int nw, int Gq,
                                                   int tid, int nt, float* dst) {
  if (tid < Gq) {
    const int h = tid;
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, pm[w * Gq + h]);
    float den = 0.f;
    for (int w = 0; w < nw; ++w) {
      const float mw = pm[w * Gq + h];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      den += pl[w * Gq + h] * f;
      pm[w * Gq + h] = f;
    }
    dst[h * (FD + 2) + FD] = M;
    dst[h * (FD + 2) + FD + 1] = den;
  }
  __syncthreads();
  for (int e = tid; e < Gq * FD; e += nt) {
    const int h = e / FD, d = e % FD;
    float num = 0.f;
    for (int w = 0; w < nw; ++w) num += part[(w * Gq + h) * FD + d] * pm[w * Gq + h];
    dst[h * (FD + 2) + d] = num;
  }
}

// final merge of ns CTA partials [ns][Gq][FD + 2] (written by other CTAs: read through L2)
__device__ __forceinline__ void attn_merge_splits(const float* sp, int ns, int Gq, int tid, int nt, float* out_u,
                                                  float* lse_u) {
  for (int e = tid; e < Gq * FD; e += nt) {
    const int h = e / FD, d = e % FD;
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) M = fmaxf(M, __ldcg(sp + (s * Gq + h) * (FD + 2) + FD));
    float num = 0.f, den = 0.f;
    for (int s = 0; s < ns; ++s) {
      const float* p = sp + (s * Gq + h) * (FD + 2);
      const float ms = __ldcg(p + FD);
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      num += __ldcg(p + d) * f;
      den += __ldcg(p + FD + 1) * f;
    }
    out_u[h * FD + d] = num / den;
    if (d == 0 && lse_u) lse_u[h] = (M + log2f(den)) * 0.6931471805599453f;
  }
}

// pad the dynamic list [n, n rounded up to 16) with token 0 (masked in attention; it keeps
// staging free of bounds checks).  Any thread may call it once n is known.
__device__ __forceinline__ void pad_dyn(int32_t* dyn, int n, int tid) {
  const int padded = (n + 15) & ~15;
  if (tid < padded - n) dyn[n + tid] = 0;
}

}  // namespace sikv

namespace sikv {

// ---------------------------------------------------------------- unit producer
// Score every prefill token of one unit and collect the top-k candidates, run by a
// 256-thread group Grp (the whole CTA, or the producer half of the persistent kernel).
//
// Selection modes: 0 nothing dynamic; 1 every candidate selected; 2 every candidate fits
// the per-warp segments (threshold -inf); 3 sampled threshold tau.  Outputs: per-warp
// candidate segments (x = key - tau, token) in cand, ms->wcnt / maxx / tau, and on return
// `fallback` = the segments are unusable (overflow or too few).  In that case the caller
// runs produce_exact().
struct UnitGeom {
  int64_t L;           // tokens this group scans (a slice of the unit for split units)
  int64_t ncand;       // selectable tokens of the whole unit (L_unit - S)
  int S, keff, mode, nchunks, capw, sstride, nsc;
  int npass;           // sample passes (long units: more sample chunks, a tighter threshold)
  int64_t flim;        // tokens below flim may be sinks
};

// Long units take up to 4 sample passes of MAX_SAMPLE_CHUNKS chunks (one per 32K tokens): the
// sampled threshold's rank error shrinks as 1/sqrt(sample), so the candidate count stays well
// inside the buffer (one pass at 128K tokens overflowed it in ~20% of units, each a rescan).
// The extra passes' keys wait for the histogram in the candidate area, past the first 512
// words (th / tmin may alias them).
constexpr int kSampleScratchWords = 512;
constexpr int kMaxSamplePasses = 4;

// sink_idx_u may be null when flim is filled in later (flim_known = 0)
__device__ __forceinline__ UnitGeom unit_geom(int64_t L, int S, int k, int capw, const int32_t* sink_idx_u,
                                              int flim_known = 1) {
  UnitGeom g;
  g.L = L;
  g.S = S;
  const int64_t ncand = L - S;
  g.ncand = ncand;
  g.keff = (int)((int64_t)k < ncand ? (int64_t)k : ncand);
  g.nchunks = (int)((L + 255) >> 8);
  g.capw = capw;
  if (g.keff == 0) g.mode = 0;
  else if (g.keff == ncand) g.mode = 1;
  else if ((int64_t)g.nchunks * 32 <= (int64_t)capw) g.mode = 2;
  else g.mode = 3;
  // a multiple of NB: every sample chunk is the first chunk of a scan batch
  g.sstride = g.mode == 3 ? (max(SSTRIDE_MIN, (g.nchunks + MAX_SAMPLE_CHUNKS - 1) / MAX_SAMPLE_CHUNKS) + NB - 1) / NB * NB
                          : 1;
  g.nsc = g.mode == 3 ? (g.nchunks + g.sstride - 1) / g.sstride : 0;
  g.npass = 1;
  if (g.mode == 3 && g.nsc == MAX_SAMPLE_CHUNKS && g.sstride >= 2 * kMaxSamplePasses) {
    const int by_len = min(kMaxSamplePasses, g.nchunks / 128);
    const int by_room = 1 + (2 * capw * DW - kSampleScratchWords) / (MAX_SAMPLE_CHUNKS * DT);
    g.npass = max(1, min(by_len, by_room));
  }
  g.flim = (S > 0 && flim_known) ? (int64_t)sink_idx_u[S - 1] + 1 : 0;
  return g;
}

__device__ __forceinline__ void load_sample(const UnitGeom& g, const uint4* signs, int tid,
                                            uint4 (&w)[MAX_SAMPLE_CHUNKS]) {
#pragma unroll
  for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
    const int64_t t = (int64_t)x * g.sstride * 256 + tid;
    w[x] = (x < g.nsc && t < g.L) ? __ldg(signs + t) : make_uint4(0, 0, 0, 0);
  }
}

// The extra sample passes of a long unit.  Keys -> xkeys[(p - 1) * 8 + x][DT]; returns the thread's count of valid keys and folds them
// into smax / smin.
template <class Key>
__device__ __forceinline__ int sample_extra_passes(const UnitGeom& g, const uint4* signs, const char* T,
                                                   const Key& lb, const uint32_t* forced, uint32_t* xkeys, int tid,
                                                   uint32_t& smax, uint32_t& smin) {
  const int off = g.sstride / g.npass;
  int nvx = 0;
  for (int p = 1; p < g.npass; ++p) {
    uint4 w[MAX_SAMPLE_CHUNKS];
#pragma unroll
    for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
      const int64_t t = ((int64_t)x * g.sstride + p * off) * 256 + tid;
      w[x] = t < g.L ? __ldg(signs + t) : make_uint4(0, 0, 0, 0);
    }
    float svx[MAX_SAMPLE_CHUNKS];
    score_batch(w, lb, T, svx);
#pragma unroll
    for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
      const int64_t t = ((int64_t)x * g.sstride + p * off) * 256 + tid;
      uint32_t key = 0;
      if (t < g.L && !(t < g.flim && forced_bit(forced, t))) key = f32_key(svx[x]);
      xkeys[((p - 1) * MAX_SAMPLE_CHUNKS + x) * DT + tid] = key;
      nvx += key != 0;
      smax = max(smax, key);
      if (key) smin = min(smin, key);
    }
  }
  return nvx;
}

// th / tmin: 256 + 256 words of scratch for the threshold histogram (may alias cand: the
// histogram is rebuilt from the register-resident sample keys for every attempt).
//
// The sampled threshold is the sample key of rank r = e + 3 sqrt(e) + 8 (e = expected
// sample items in the top-k).  When the scan then overflows a warp segment (tau too low) or
// yields fewer than k candidates (tau too high), r is rescaled from the observed counts and
// the scan is repeated (at most kRetries times) before falling back to the exact path.
constexpr int kRetries = 2;
constexpr double kTauSig = 3.0, kTauAdd = 8.0;   // sample-rank margin: r = e + SIG sqrt(e) + ADD

// XP: the unit may take extra sample passes (g.npass > 1; instantiated for long units only,
// so the short-unit kernels keep their register allocation)
template <class Grp, class Xch = NoX, class Key = RepKey, int NBT = NB, bool XP = false>
__device__ __forceinline__ bool produce_candidates(const UnitGeom& g, const uint4* signs, const char* T,
                                                   const uint32_t* forced, const uint4 (&wsamp)[MAX_SAMPLE_CHUNKS],
                                                   uint32_t* cand, int* th, uint32_t* tmin, Misc* ms,
                                                   uint32_t& tau_out, const Xch& xch = Xch(),
                                                   long long* prof = nullptr) {
  const int tid = Grp::tid(), lane = tid & 31, warp = tid >> 5;
  const Key lb(lane);
  const int capw = g.capw;
  uint32_t* seg = cand + 2 * warp * capw;
  uint32_t sk[MAX_SAMPLE_CHUNKS];
  int nsv = 0, nsv0 = 0, r = 0;     // sample keys (all passes / the first pass), sample rank
  uint32_t kmx = 0, kmn = 0;
  if (tid == 0) { ms->maxx = 0; ms->bad = 0; }
  if (g.mode == 3) {
    // ---------------- B1: score the sample chunks (kept in registers)
    float sv[MAX_SAMPLE_CHUNKS];
    score_batch(wsamp, lb, T, sv);
    int nv = 0;
    uint32_t smax = 0, smin = 0xFFFFFFFFu;
#pragma unroll
    for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
      const int64_t t = (int64_t)x * g.sstride * 256 + tid;
      uint32_t key = 0;
      if (x < g.nsc && t < g.L && !(t < g.flim && forced_bit(forced, t))) key = f32_key(sv[x]);
      sk[x] = key;
      nv += key != 0;
      smax = max(smax, key);
      if (key) smin = min(smin, key);
    }
    nv = warp_sum(nv);
    // extra passes (long units): chunks offset by p * sstride / npass from the first pass's,
    // rescored by the scan (not skipped); keys to the scratch words for the histogram
    int nvx = 0;
    if constexpr (XP)
      if (g.npass > 1)
        nvx = warp_sum(sample_extra_passes(g, signs, T, lb, forced, cand + kSampleScratchWords, tid, smax, smin));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
      smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
    }
    if (tid == 0) { ms->nsv = 0; if (XP) ms->total = 0; ms->tau = 0xFFFFFFFFu; }
    Grp::sync();
    if (lane == 0) {
      atomicAdd(&ms->nsv, nv);
      if (XP && nvx) atomicAdd(&ms->total, nvx);
      atomicMax(&ms->maxx, smax);
      atomicMin(&ms->tau, smin);
    }
    Grp::sync();
    nsv = ms->nsv;
    nsv0 = nsv;
    if constexpr (XP) nsv += ms->total;
    kmx = ms->maxx;
    kmn = ms->tau;
    xch.sample(nsv, kmx, kmn);            // cluster: the whole unit's sample
    if (prof && tid == 0) prof[7] = clock64();            // sample scored
    const double e = (double)g.keff * (double)nsv / (double)(g.ncand);
    r = min((int)ceil(e + kTauSig * sqrt(e) + kTauAdd), nsv);
  }
  const float fmn = __uint_as_float(unkey_bits(kmn)), fmx = __uint_as_float(unkey_bits(kmx));
  const float scale = fmx > fmn ? 256.0f / (fmx - fmn) : 0.f;
  const int Li = (int)g.L;
  const int end_s = g.nsc * g.sstride;
  const uint4* pbase = signs + tid;
  asm volatile("" : "+l"(pbase));   // kept in registers, not rematerialised from the arguments per batch
  const uint64_t pol = l2_evict_first_policy();
  auto load_batch = [&](int c0, uint4 (&w)[NBT]) {
    const uint4* p = pbase + (int64_t)c0 * 256;     // constant offsets 4 KiB apart: no per-load address math
    if ((c0 + NBT) * 256 <= Li) {
#pragma unroll
      for (int x = 0; x < NBT; ++x) w[x] = ld_stream(p + 256 * x, pol);
    } else {
      const int t0 = c0 * 256 + tid;
#pragma unroll
      for (int x = 0; x < NBT; ++x) w[x] = t0 + 256 * x < Li ? ld_stream(p + 256 * x, pol) : make_uint4(0, 0, 0, 0);
    }
  };
  for (int attempt = 0;; ++attempt) {
    int wc = 0;
    uint32_t mx = 0;
    uint32_t tau = 1;
    if (g.mode == 3) {
      if (r >= 1) {
        // threshold histogram of the sample keys (256 value bins), rank r from the top
        for (int i = tid; i < 256; i += DT) { th[i] = 0; tmin[i] = 0xFFFFFFFFu; }
        Grp::sync();
#pragma unroll
        for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
          const uint32_t kx = sk[x];
          if (kx) {
            const int b = min(255, (int)((__uint_as_float(unkey_bits(kx)) - fmn) * scale));
            atomicAdd(&th[b], 1);
            atomicMin(&tmin[b], kx);
          }
        }
        if (XP && attempt == 0 && g.npass > 1) {   // the scan overwrites the scratch: first attempt only
          const uint32_t* xkeys = cand + kSampleScratchWords;
          for (int i = tid; i < (g.npass - 1) * MAX_SAMPLE_CHUNKS * DT; i += DT) {
            const uint32_t kx = xkeys[i];
            if (kx) {
              const int b = max(0, min(255, (int)((__uint_as_float(unkey_bits(kx)) - fmn) * scale)));
              atomicAdd(&th[b], 1);
              atomicMin(&tmin[b], kx);
            }
          }
        }
        Grp::sync();
        const int* thm = th;
        const uint32_t* tminm = tmin;
        xch.hist256(thm, tminm);              // cluster: merged over the CTAs
        if (warp == 0) {
          int loc[8], s8 = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) { loc[i] = thm[255 - 8 * lane - i]; s8 += loc[i]; }
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
        Grp::sync();
        tau = tminm[ms->digit];         // smallest sample key in the boundary bin
        if (prof && tid == 0 && attempt == 0) prof[8] = clock64();   // threshold known
      }
      Grp::sync();
      if (tid == 0) { ms->maxx = 0; ms->bad = 0; }
      Grp::sync();
      uint32_t bits = 0, skx[MAX_SAMPLE_CHUNKS];
#pragma unroll
      for (int x = 0; x < MAX_SAMPLE_CHUNKS; ++x) {
        skx[x] = sk[x];
        if (x < g.nsc && skx[x] != 0 && skx[x] >= tau) bits |= 1u << x;
      }
      const int cnt = __popc(bits);
      int inc = cnt;
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
          const uint32_t xk = skx[x] - tau;
          if (pos < capw) { seg[2 * pos] = xk; seg[2 * pos + 1] = (uint32_t)(x * g.sstride * 256 + tid); }
          mx = max(mx, xk);
          ++pos;
        }
      }
    }
    // ---------------- B2: score everything else, keep score >= tau (compared as floats)
    const float tauf = g.mode == 2 ? -INFINITY : __uint_as_float(unkey_bits(tau));
    int next_s = g.mode == 3 ? 0 : 0x7fffffff;      // next sample chunk (already scored in B1)
    const uint32_t segs = (uint32_t)__cvta_generic_to_shared(seg);
    // register double buffer: the loads of batch c0 + NB are in flight while batch c0 scores
    uint4 wn[NBT];
    load_batch(0, wn);
    for (int c0 = 0; c0 < g.nchunks; c0 += NBT) {
      // sample chunks (scored in B1) open their batch (g.sstride is a multiple of NBT)
      const uint32_t xsm = c0 == next_s && c0 < end_s ? 1u : 0u;
      if (xsm) next_s += g.sstride;
      const int t0 = c0 * 256 + tid;
      const bool full = (c0 + NBT) * 256 <= Li;
      uint4 w[NBT];
#pragma unroll
      for (int x = 0; x < NBT; ++x) w[x] = wn[x];
      if (c0 + NBT < g.nchunks) load_batch(c0 + NBT, wn);
      float sv[NBT];
      score_batch(w, lb, T, sv);
      uint32_t bits = 0;
#pragma unroll
      for (int x = 0; x < NBT; ++x)
        if (sv[x] >= tauf) bits |= 1u << x;
      bits &= ~xsm;
      if (!full) bits &= (Li - t0 > 0) ? ((Li - t0 + 255) / 256 >= NBT ? 0xFFu : ((1u << ((Li - t0 + 255) / 256)) - 1u)) : 0u;
      if (c0 * 256 < g.flim) {
#pragma unroll
        for (int x = 0; x < NBT; ++x)
          if (t0 + 256 * x < Li && forced_bit(forced, t0 + 256 * x)) bits &= ~(1u << x);
      }
      // warp-compacted append: one scan per batch
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
        const uint32_t xk = f32_key_fast(pick_dyn<NBT>(sv, x)) - tau;
        st_shared_v2_if(pos < capw, segs + 8u * (uint32_t)pos, xk, (uint32_t)(t0 + 256 * x));
        mx = max(mx, xk);
        ++pos;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) { ms->wcnt[warp] = wc; atomicMax(&ms->maxx, mx); if (wc > capw) ms->bad = 1; }
    Grp::sync();
    int total = 0, maxwc = 0;
    for (int w2 = 0; w2 < DW; ++w2) { total += ms->wcnt[w2]; maxwc = max(maxwc, ms->wcnt[w2]); }
    tau_out = tau;
    bool bad = ms->bad != 0;
    xch.counts(total, maxwc, bad);        // cluster: unit totals, any CTA overflowing
    if (prof && tid == 0) { prof[9] = attempt; prof[10] = total; prof[11] = maxwc; }
    if (!bad && total >= g.keff) return false;
    if (g.mode != 3 || attempt >= kRetries || r < 1) return true;
    // rescale the sample rank from the observed candidate counts and scan again
    int r2 = bad ? (int)((double)r * 0.85 * (double)capw / (double)maxwc)
                 : min(nsv, (int)ceil((double)r * 1.25 * (double)g.keff / (double)max(total, 1)) + 8);
    if (r2 < 1 || r2 == r) return true;
    if (XP && attempt == 0 && nsv0 < nsv) {      // retries rank the first pass's keys only
      r2 = max(1, min(nsv0, (int)((double)r2 * (double)nsv0 / (double)nsv + 0.5)));
      nsv = nsv0;
    }
    r = r2;
    Grp::sync();                          // every thread has read ms before it is reset
  }
}

// Exact fallback: multi-pass radix select over rescored keys, then gt / eq bitmaps (zeroed
// here; smem or global) of key > K* and key == K*.  hist needs NBIN + 33 ints.
template <class Grp, class Xch = NoX, class Key = RepKey, int NBINT = NBIN>
__device__ __forceinline__ void produce_exact(const UnitGeom& g, const uint4* signs, const char* T,
                                              const uint32_t* forced, int* hist, Misc* ms, uint32_t* gt,
                                              uint32_t* eq, uint32_t& kstar, int& need_eq, int& eq_count,
                                              const Xch& xch = Xch()) {
  const int tid = Grp::tid(), lane = tid & 31;
  const Key lb(lane);
  const int64_t L = g.L;
  const int nchunks = g.nchunks;
  radix_kth<Grp, Xch, NBINT>([&](auto f) {
    for (int c = 0; c < nchunks; ++c) {
      const int64_t t = (int64_t)c * 256 + tid;
      if (t < L && !forced_bit(forced, t)) f(f32_key(score_token(__ldg(signs + t), lb, T)));
    }
  }, 0xFFFFFFFFu, g.keff, hist, ms, kstar, need_eq, xch);
  const int W = (int)((L + 31) >> 5);
  for (int i = tid; i < 2 * W; i += DT) (i < W ? gt[i] : eq[i - W]) = 0u;
  if (tid == 0) ms->nsv = 0;
  __threadfence();
  Grp::sync();
  for (int c = 0; c < nchunks; ++c) {
    const int64_t t = (int64_t)c * 256 + tid;
    if (t < L && !forced_bit(forced, t)) {
      const uint32_t key = f32_key(score_token(__ldg(signs + t), lb, T));
      if (key > kstar) atomicOr(&gt[t >> 5], 1u << (t & 31));
      else if (key == kstar) { atomicOr(&eq[t >> 5], 1u << (t & 31)); atomicAdd(&ms->nsv, 1); }
    }
  }
  __threadfence();
  Grp::sync();
  eq_count = ms->nsv;
}

// Exact k-th key among the candidate segments: xk (relative to tau) and how many of the
// items equal to it belong to the top keff.
template <class Grp, class Xch = NoX, int NBINT = NBIN>
__device__ __forceinline__ void kth_from_candidates(const UnitGeom& g, const uint32_t* cand, const int* wcnt,
                                                    uint32_t maxx, int* hist, Misc* ms, uint32_t& xk,
                                                    int& need_eq, const Xch& xch = Xch()) {
  const int tid = Grp::tid(), lane = tid & 31, warp = tid >> 5;
  const uint32_t* seg = cand + 2 * warp * g.capw;
  const int n = wcnt[warp];
  maxx = xch.maxu(maxx);
  radix_kth<Grp, Xch, NBINT>([&](auto f) {
    for (int i = lane; i < n; i += 32) f(seg[2 * i]);
  }, maxx, g.keff, hist, ms, xk, need_eq, xch);
}

// gt / eq bitmaps (zeroed here) of the candidates above / at the k-th key xk
template <class Grp>
__device__ __forceinline__ void bitmaps_from_candidates(const UnitGeom& g, const uint32_t* cand, const int* wcnt,
                                                        uint32_t xk, Misc* ms, uint32_t* gt, uint32_t* eq,
                                                        int& eq_count) {
  const int tid = Grp::tid(), lane = tid & 31, warp = tid >> 5;
  const uint32_t* seg = cand + 2 * warp * g.capw;
  const int n = wcnt[warp];
  const int W = (int)((g.L + 31) >> 5);
  for (int i = tid; i < W; i += DT) { gt[i] = 0u; eq[i] = 0u; }
  if (tid == 0) ms->nsv = 0;
  Grp::sync();
  for (int i = lane; i < n; i += 32) {
    const uint32_t x = seg[2 * i], t = seg[2 * i + 1];
    if (x > xk) atomicOr(&gt[t >> 5], 1u << (t & 31));
    else if (x == xk) { atomicOr(&eq[t >> 5], 1u << (t & 31)); atomicAdd(&ms->nsv, 1); }
  }
  Grp::sync();
  eq_count = ms->nsv;
}

// Exact k-th key among the candidate segments, then the gt / eq bitmaps (zeroed here).
template <class Grp, class Xch = NoX, int NBINT = NBIN>
__device__ __forceinline__ void select_from_candidates(const UnitGeom& g, const uint32_t* cand, const int* wcnt,
                                                       uint32_t maxx, uint32_t tau, int* hist, Misc* ms,
                                                       uint32_t* gt, uint32_t* eq, uint32_t& kstar,
                                                       int& need_eq, int& eq_count, const Xch& xch = Xch()) {
  uint32_t xk;
  kth_from_candidates<Grp, Xch, NBINT>(g, cand, wcnt, maxx, hist, ms, xk, need_eq, xch);
  kstar = xk + tau;
  bitmaps_from_candidates<Grp>(g, cand, wcnt, xk, ms, gt, eq, eq_count);
}

// The dynamic list straight from the candidate segments, without bitmaps: every candidate
// with x > xk plus the ties x == xk, in segment order (warp 0's segment first, each in
// scan order — deterministic).  Valid only when every tie is taken; returns -1 when the
// ties must be cut by token index (the caller then takes the bitmap path).
template <class Grp>
__device__ __forceinline__ int emit_from_segments(const UnitGeom& g, const uint32_t* cand, const int* wcnt,
                                                  uint32_t xk, int need_eq, int32_t* dyn, Misc* ms) {
  const int tid = Grp::tid(), lane = tid & 31, warp = tid >> 5;
  const uint32_t* seg = cand + 2 * warp * g.capw;
  const int n = wcnt[warp];
  int ngt = 0, neq = 0;
  for (int i = lane; i < n; i += 32) {
    const uint32_t x = seg[2 * i];
    ngt += x > xk;
    neq += x == xk;
  }
  ngt = warp_sum(ngt);
  neq = warp_sum(neq);
  int pos, epos, tot, etot;
  block_exscan2<Grp>(lane == 0 ? ngt + neq : 0, lane == 0 ? neq : 0, pos, epos, tot, etot, ms->wsum);
  if (etot != need_eq) return -1;
  pad_dyn(dyn, tot, tid);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    const bool take = i < n && seg[2 * i] >= xk;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) dyn[pos + __popc(m & ((1u << lane) - 1u))] = (int32_t)seg[2 * i + 1];
    pos += __popc(m);
  }
  Grp::sync();
  return tot;
}

// Ordered emission: dynamic list (smem, nullable) and the sorted selection (global, nullable).
// Returns the dynamic count.
template <class Grp>
__device__ __forceinline__ int emit_selection(const UnitGeom& g, int mode, const uint32_t* forced,
                                              const uint32_t* gt, const uint32_t* eq, int need_eq, int eq_count,
                                              int32_t* dyn, int32_t* sel_u, int R, int32_t* sel_count_u,
                                              Misc* ms) {
  const int tid = Grp::tid();
  const int64_t L = g.L;
  const int W = (int)((L + 31) >> 5);
  const int per = (W + DT - 1) / DT;
  const int w0 = tid * per, w1 = min(W, w0 + per);
  // ties at the k-th key: keep the lowest-index need_eq of them (prefix over the eq bitmap);
  // when every tie is taken (the usual case) no prefix is needed
  const bool all_eq = mode < 2 || eq_count == need_eq;
  int eq_before = 0;
  if (!all_eq) {
    int my_eq = 0;
    for (int x = w0; x < w1; ++x) my_eq += __popc(eq[x]);
    int dummy, t1, t2;
    block_exscan2<Grp>(my_eq, 0, eq_before, dummy, t1, t2, ms->wsum);
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
  block_exscan2<Grp>(nd, nsl, dpos, spos, dtot, stot, ms->wsum);
  if (dyn) pad_dyn(dyn, dtot, tid);
  eb = eq_before;
  for (int x = w0; x < w1; ++x) {
    uint32_t d = dbits(x, eb);
    uint32_t sb = d | forced[x];
    if (dyn)
      while (d) { const int b = __ffs(d) - 1; d &= d - 1; dyn[dpos++] = x * 32 + b; }
    if (sel_u)
      while (sb) { const int b = __ffs(sb) - 1; sb &= sb - 1; sel_u[spos++] = x * 32 + b; }
  }
  if (sel_u)
    for (int r = tid; r < R; r += DT) sel_u[stot + r] = (int32_t)(L + r);
  if (tid == 0 && sel_count_u) *sel_count_u = stot + R;
  Grp::sync();
  return dtot;
}

// Select + emit for a unit whose candidates sit in per-warp segments (mode >= 2, no
// fallback): the exact k-th key, then the dynamic list from the segments.  The sorted
// selection (sel_u / sel_count_u, optional) and the rare index-cut ties go through the
// bitmaps.  Returns the dynamic count; kstar = absolute k-th key.
template <class Grp, int NBINT = NBIN>
__device__ __forceinline__ int select_emit_candidates(const UnitGeom& g, const uint32_t* forced, const uint32_t* cand,
                                                      const int* wcnt, uint32_t maxx, uint32_t tau, int* hist,
                                                      Misc* ms, uint32_t* gt, uint32_t* eq, int32_t* dyn,
                                                      int32_t* sel_u, int R, int32_t* sel_count_u, uint32_t& kstar,
                                                      long long* prof = nullptr) {
  uint32_t xk;
  int need_eq;
  kth_from_candidates<Grp, NoX, NBINT>(g, cand, wcnt, maxx, hist, ms, xk, need_eq);
  if (prof && Grp::tid() == 0) prof[12] = clock64();
  kstar = xk + tau;
  int ndyn = emit_from_segments<Grp>(g, cand, wcnt, xk, need_eq, dyn, ms);
  if (prof && Grp::tid() == 0) prof[13] = clock64();
  if (ndyn < 0 || sel_u || sel_count_u) {
    int eq_count;
    bitmaps_from_candidates<Grp>(g, cand, wcnt, xk, ms, gt, eq, eq_count);
    const int nd = emit_selection<Grp>(g, g.mode, forced, gt, eq, need_eq, eq_count, ndyn < 0 ? dyn : nullptr,
                                       sel_u, R, sel_count_u, ms);
    if (ndyn < 0) ndyn = nd;
  }
  return ndyn;
}

}  // namespace sikv
