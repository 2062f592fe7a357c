// Shared device helpers for the self-indexing KV-cache kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sikv {

// ------------------------------------------------------------------ input dtypes
enum InDType : int { IN_F32 = 0, IN_F64 = 1, IN_BF16 = 2 };

__device__ __forceinline__ double load_in(const void* p, int dt, int64_t i) {
  if (dt == IN_F64) return reinterpret_cast<const double*>(p)[i];
  if (dt == IN_F32) return (double)reinterpret_cast<const float*>(p)[i];
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

// ------------------------------------------------------------------ order-preserving keys
// float -> uint32 with the same ordering; -0.0 is canonicalised to +0.0 first so
// that ties between -0 and +0 break by index exactly like numpy's stable argsort.
__device__ __forceinline__ uint32_t f32_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t f64_key(double f) {
  uint64_t u = (uint64_t)__double_as_longlong(f);
  if (u == 0x8000000000000000ull) u = 0ull;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// ------------------------------------------------------------------ fast-layout constants
// D = 128 channels, 32 sign groups (16 packed bytes), 4 quant groups of 32 channels.
constexpr int FD = 128;
constexpr int FSIGN = 16;      // bytes per token in the sign plane
constexpr int FREC = 128;      // bytes per token record
// record byte offsets
constexpr int R_K4 = 0;        // 64 B K as e2m1 nibbles (sign | 2-bit code), MMA-permuted
constexpr int R_VPAY = 64;     // 32 B V payload, MMA-permuted
constexpr int R_KPAR = 96;     // 4 x (2 qs, zp) fp16
constexpr int R_VPAR = 112;    // 4 x (qs, zp) fp16
// 16-bit records (the bits = 16 "Ours (16 bits)" variant, cache.py:236-238 at model precision):
// 512 B per token.  Bytes 0-255: K^ = K' / alpha-hat in fp16, B-operand order: 64-B chunk t4
// holds, as word 2s + e, channels (16 s + 8 e + 2 t4, +1) (one quad lane's 8 k-steps).  Bytes
// 256-511: V in fp16, 32-B chunk g holds, as word m, channels (16 m + g, 16 m + g + 8) (the
// A-operand rows of lane group g for the 8 m-tiles).
constexpr int FREC16 = 512;
__host__ __device__ __forceinline__ int k16_off(int ch) {   // byte offset of K channel ch
  const int s = ch >> 4, e = (ch >> 3) & 1, t4 = (ch & 7) >> 1;
  return 64 * t4 + 4 * (2 * s + e) + 2 * (ch & 1);
}
__host__ __device__ __forceinline__ int v16_off(int ch) {   // byte offset of V channel ch
  const int m = ch >> 4, r = ch & 15;
  return 256 + 32 * (r & 7) + 4 * m + 2 * (r >> 3);
}
// staged 16-bit block: 16-B unit u of block token j at unit u ^ sw16(j, u) (conflict-free
// K and V fragment reads; found by exhaustive search over XOR swizzles)
__host__ __device__ __forceinline__ int sw16(int j, int u) {
  return u ^ (((u >> 3) ^ ((j & 1) << 1) ^ ((j >> 1) & 1) ^ (((j >> 2) & 1) << 2)) & 7);
}

// one 16-row block of forced rows (sinks, then recents): K^ fragments [32 lanes][32 words],
// V fragments [32 lanes][32 words], then 16 float32 row scales (a power of two per row:
// K^ = K' / (alpha-hat * scale) stays within fp16 for recent rows whose |K'| exceeds the
// prefill alpha; the logit is multiplied back by the scale)
constexpr int FBLK_WORDS = 2 * 32 * 32 + 32;   // scales padded to a 128-B line: blocks stay line-aligned

// ---- K nibble permutation (B operand of q~ K^T, m16n8k16, one token per n column).
// A nibble is an e2m1 value: bit 3 = sign of K' (1 = negative), bits 0-1 = the 2-bit
// magnitude code c, bit 2 = 0, so it decodes (cvt.rn.f16x2.e2m1x2) to sign * c / 2 and
// K^ = (2 qs) x + copysign(zp, x).  Thread t4 of a quad owns the 16-byte chunk t4 (words
// 4 t4 .. 4 t4 + 3); byte 2s + e of the chunk holds channels 16s + 8e + 2t4 (lo nibble) and
// +1 (hi nibble).  Group j's channels fill exactly word 4 t4 + j.
__host__ __device__ __forceinline__ void k4_pos(int ch, int& word, int& bit) {
  const int j = ch >> 5, n = ch & 31;
  const int ss = n >> 4, e = (n >> 3) & 1, rr = n & 7;
  word = 4 * (rr >> 1) + j;
  bit = 16 * ss + 8 * e + 4 * (rr & 1);
}
// ---- V payload permutation (A operand of V^T P^T, m16n8k16, one channel per m row)
// word g (0..7) holds channels 16m + g + 8e (m = 0..7, e = 0,1):
// byte j = m>>1, bits [2i', 2i'+2) with i' = 2*(m&1) + e.
__host__ __device__ __forceinline__ void vpay_pos(int ch, int& word, int& bit) {
  int m = ch >> 4, r = ch & 15;
  int g = r & 7, e = r >> 3;
  word = g;
  bit = 8 * (m >> 1) + 2 * (2 * (m & 1) + e);
}

// ------------------------------------------------------------------ warp helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ mma.sync m16n8k16 f16 -> f32
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 8x8 b16 transpose across the warp: the thread holding (row g, cols 2t4, 2t4 + 1) of the
// input receives (row g, cols 2t4, 2t4 + 1) of the transpose
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  // (a & mask) | magic
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(magic));
  return r;
}
__device__ __forceinline__ uint32_t lop3_xor_and(uint32_t v, uint32_t s, uint32_t mask) {
  // v ^ (s & mask)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(v), "r"(s), "r"(mask));
  return r;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

}  // namespace sikv
