// Prefill-side key/value compression (encoder), float64-exact against the reference.
//
//   K1 stats_partial / stats_final : mu, alpha per (unit, channel)     normalize.py:56-61
//   K2 pack                        : sign codes, B-bit payloads,        codebook.py:116-125,
//                                    fp16 params, codebook partials     quantizer.py:97-170
//   K3 codebook_final              : centroid means                     codebook.py:128-160
//   row gather / append            : full-precision sink / recent rows  cache.py:247-287
//
// Exactness argument for mu: the reference sums rows sequentially in float64.  For each
// channel we also compute sum|x| and the lowest set-bit exponent e_low over all values.
// Every partial sum of any subset is a multiple of 2^e_low bounded by sum|x|; if
// sum|x| < 2^(e_low+52) every partial sum is exactly representable, so any summation
// order (here: per-split then fixed-order combine) yields the reference's bits.  Channels
// failing this certificate are re-summed sequentially in row order (reference order).
#include "common.cuh"
#include <math.h>
#include <type_traits>

namespace sikv {

__device__ __forceinline__ int lowbit_exp(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7FF);
  uint64_t m = b & ((1ull << 52) - 1);
  if (e == 0) {
    if (m == 0) return 0x7fffffff;
    return -1074 + __ffsll((long long)m) - 1;
  }
  m |= (1ull << 52);
  return e - 1075 + __ffsll((long long)m) - 1;
}

// ---------------------------------------------------------------- K1: channel statistics
__global__ void stats_partial_kernel(const void* __restrict__ keys, int dt, int64_t L, int D,
                                     int nsplit, double* __restrict__ part, int* __restrict__ status) {
  const int u = blockIdx.x, s = blockIdx.y;
  const int64_t per = (L + nsplit - 1) / nsplit;
  const int64_t t0 = s * per, t1 = min(L, t0 + per);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double sum = -0.0, sab = 0.0, mn = INFINITY, mx = -INFINITY;
    int low = 0x7fffffff;
    bool bad = false;
    const int64_t base = (int64_t)u * L * D + c;
    for (int64_t t = t0; t < t1; ++t) {
      double x = load_in(keys, dt, base + t * D);
      bad |= !isfinite(x);
      sum += x;
      sab += fabs(x);
      mn = fmin(mn, x);
      mx = fmax(mx, x);
      if (x != 0.0) low = min(low, lowbit_exp(x));
    }
    if (bad) atomicOr(status, 4);
    double* p = part + (((int64_t)u * nsplit + s) * D + c) * 5;
    p[0] = sum; p[1] = sab; p[2] = mn; p[3] = mx; p[4] = __longlong_as_double((long long)low);
  }
}

// One warp per (unit, channel): lanes combine the split partials (exact under the
// certificate, so the combine order is free), lane 0 finalises.
__global__ void __launch_bounds__(256) stats_final_kernel(const void* __restrict__ keys, int dt, int64_t L, int D,
                                                          int nsplit, const double* __restrict__ part,
                                                          double* __restrict__ mu64, double* __restrict__ alpha64,
                                                          float* __restrict__ mu32, float* __restrict__ alpha32,
                                                          int* __restrict__ status) {
  const int u = blockIdx.x, lane = threadIdx.x & 31;
  const int c = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (c >= D) return;
  double sum = -0.0, sab = 0.0, mn = INFINITY, mx = -INFINITY;
  int low = 0x7fffffff;
  for (int s = lane; s < nsplit; s += 32) {
    const double* p = part + (((int64_t)u * nsplit + s) * D + c) * 5;
    sum += p[0]; sab += p[1]; mn = fmin(mn, p[2]); mx = fmax(mx, p[3]);
    low = min(low, (int)__double_as_longlong(p[4]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    sab += __shfl_xor_sync(0xffffffffu, sab, o);
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    low = min(low, __shfl_xor_sync(0xffffffffu, low, o));
  }
  if (lane) return;
  sab *= 1.0 + 0x1p-40;                          // covers the rounding of the combine
  const bool exact = (low == 0x7fffffff) || (low + 52 < 1023 && sab < ldexp(1.0, low + 52));
  if (!exact) {
    // certificate failed: replay the reference's sequential row order (loads batched ahead)
    atomicOr(status, 8);
    const int64_t base = (int64_t)u * L * D + c;
    sum = load_in(keys, dt, base);
    int64_t t = 1;
    constexpr int RU = 16;
    for (; t + RU <= L; t += RU) {
      double v[RU];
#pragma unroll
      for (int k = 0; k < RU; ++k) v[k] = load_in(keys, dt, base + (t + k) * D);
#pragma unroll
      for (int k = 0; k < RU; ++k) sum += v[k];
    }
    for (; t < L; ++t) sum += load_in(keys, dt, base + t * D);
  }
  const double mu = sum / (double)L;
  const double a = fmax(fabs(mx - mu), fabs(mn - mu));
  mu64[(int64_t)u * D + c] = mu;
  alpha64[(int64_t)u * D + c] = a;
  if (mu32) mu32[(int64_t)u * D + c] = (float)mu;
  if (alpha32) alpha32[(int64_t)u * D + c] = (float)a;
}


// Vectorised statistics for bf16 / f32 inputs: lane l owns channels 4l..4l+3, the 8 warps
// take interleaved rows; warp partials combine in fixed order (the sums are exact under the
// certificate, so the order does not matter; otherwise stats_final replays the row order).
__device__ __forceinline__ int lowbit_f32(float x) {
  const uint32_t b = __float_as_uint(x);
  const int e = (int)((b >> 23) & 0xFF);
  const uint32_t m = b & 0x7FFFFFu;
  if (e == 0) return m ? -149 + __ffs((int)m) - 1 : 0x7fffffff;
  return e - 150 + __ffs((int)(m | 0x800000u)) - 1;
}

template <int DTY>
__device__ __forceinline__ void load4(const void* p, int64_t idx, float (&x)[4]) {
  if (DTY == IN_BF16) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p) + idx));
    x[0] = __uint_as_float(w.x << 16); x[1] = __uint_as_float(w.x & 0xFFFF0000u);
    x[2] = __uint_as_float(w.y << 16); x[3] = __uint_as_float(w.y & 0xFFFF0000u);
  } else {
    const float4 w = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + idx));
    x[0] = w.x; x[1] = w.y; x[2] = w.z; x[3] = w.w;
  }
}

template <int DTY>
__global__ void __launch_bounds__(256) stats_partial_fast_kernel(const void* __restrict__ keys, int64_t L, int D,
                                                                 int nsplit, double* __restrict__ part,
                                                                 int* __restrict__ status) {
  __shared__ double red[8][128][5];
  const int u = blockIdx.x, s = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (L + nsplit - 1) / nsplit;
  const int64_t t0 = s * per, t1 = min(L, t0 + per);
  const bool active = 4 * lane < D;
  // sum: exact float64 (certificate in stats_final); sab: float32 rounded up, an upper bound
  // on sum|x|; low: lowest set-bit exponent (bf16: a lower bound from the exponent field)
  double sum[4] = {-0.0, -0.0, -0.0, -0.0};
  float sab[4] = {0.f, 0.f, 0.f, 0.f};
  float mn[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  int low[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
  uint32_t emin[4] = {0x7F800000u, 0x7F800000u, 0x7F800000u, 0x7F800000u};
  if (active) {
    constexpr int UN = 8;                        // rows per warp per batch; two batches in flight
    using Raw = typename std::conditional<DTY == IN_BF16, uint2, float4>::type;
    auto ld = [&](int64_t t) -> Raw {
      if (t >= t1) {                             // -0 leaves sum / sab / low unchanged
        if constexpr (DTY == IN_BF16) return make_uint2(0x80008000u, 0x80008000u);
        else return make_float4(-0.f, -0.f, -0.f, -0.f);
      }
      const int64_t idx = ((int64_t)u * L + t) * D + 4 * lane;
      if constexpr (DTY == IN_BF16)
        return __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(keys) + idx));
      else
        return __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(keys) + idx));
    };
    Raw nx[UN];
#pragma unroll
    for (int r = 0; r < UN; ++r) nx[r] = ld(t0 + warp + 8 * r);
    for (int64_t tb = t0 + warp; tb < t1; tb += 8 * UN) {
      float x[UN][4];
#pragma unroll
      for (int r = 0; r < UN; ++r) {
        if constexpr (DTY == IN_BF16) {
          x[r][0] = __uint_as_float(nx[r].x << 16); x[r][1] = __uint_as_float(nx[r].x & 0xFFFF0000u);
          x[r][2] = __uint_as_float(nx[r].y << 16); x[r][3] = __uint_as_float(nx[r].y & 0xFFFF0000u);
        } else {
          x[r][0] = nx[r].x; x[r][1] = nx[r].y; x[r][2] = nx[r].z; x[r][3] = nx[r].w;
        }
      }
      if (tb + 8 * UN < t1) {                    // the next batch's loads fly while this one sums
#pragma unroll
        for (int r = 0; r < UN; ++r) nx[r] = ld(tb + 8 * UN + 8 * r);
      }
#pragma unroll
      for (int r = 0; r < UN; ++r) {
        const bool in = tb + 8 * r < t1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float v = x[r][i];
          sum[i] += (double)v;
          sab[i] = __fadd_ru(sab[i], fabsf(v));
          if (in) { mn[i] = fminf(mn[i], v); mx[i] = fmaxf(mx[i], v); }
          if (DTY == IN_BF16) {
            const uint32_t eb = __float_as_uint(v) & 0x7F800000u;
            emin[i] = min(emin[i], v != 0.f ? eb : 0x7F800000u);
          } else if (v != 0.f) {
            low[i] = min(low[i], lowbit_f32(v));
          }
        }
      }
    }
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      bad |= !isfinite(sum[i]) || mx[i] == INFINITY || mn[i] == -INFINITY;
      // bf16 values are multiples of 2^(e - 134) (normal, biased exponent e) or 2^-133
      if (DTY == IN_BF16 && emin[i] != 0x7F800000u) low[i] = emin[i] ? (int)(emin[i] >> 23) - 134 : -133;
      double* r = red[warp][4 * lane + i];
      r[0] = sum[i]; r[1] = (double)sab[i]; r[2] = mn[i]; r[3] = mx[i]; r[4] = __longlong_as_double((long long)low[i]);
    }
    if (bad) atomicOr(status, 4);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += 256) {
    double a0 = -0.0, a1 = 0.0, a2 = INFINITY, a3 = -INFINITY;
    int lo = 0x7fffffff;
    for (int w = 0; w < 8; ++w) {
      a0 += red[w][c][0]; a1 += red[w][c][1]; a2 = fmin(a2, red[w][c][2]); a3 = fmax(a3, red[w][c][3]);
      lo = min(lo, (int)__double_as_longlong(red[w][c][4]));
    }
    double* p = part + (((int64_t)u * nsplit + s) * D + c) * 5;
    p[0] = a0; p[1] = a1 * (1.0 + 0x1p-40); p[2] = a2; p[3] = a3; p[4] = __longlong_as_double((long long)lo);
  }
}

// ---------------------------------------------------------------- K2: pack
struct PackArgs {
  const void* keys; const void* values; int dt;
  int64_t L; int D; int bits; int gs; int siq;
  const double* mu64; const double* alpha64;
  // reference layout (nullable)
  uint8_t* codes_ref; uint8_t* kq_ref; __half* ks_ref; __half* kz_ref;
  uint8_t* vq_ref; __half* vs_ref; __half* vz_ref;
  // fast layout (nullable)
  uint8_t* signs_fast; uint8_t* recs_fast;
  // codebook partials
  double* cb_part; int* cb_cnt; int ntiles; int tile;
  int* status;
  const uint8_t* codes_in;   // optional externally supplied sign codes (reference layout)
};

constexpr int PACK_WARPS = 4;

// min/max over the lanes of one quantisation group (lanes_per_group is a power of two)
__device__ __forceinline__ void group_minmax(double& mn, double& mx, int lpg) {
  for (int o = 1; o < lpg; o <<= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
}

// quantizer.py:119-130 on one lane's 4 elements; returns the 4 codes and the fp16 params
__device__ __forceinline__ void quant4(const double (&x)[4], bool active, int lpg, int levels,
                                       uint32_t (&code)[4], __half& qs16, __half& zp16, int* status) {
  double mn = INFINITY, mx = -INFINITY;
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { mn = fmin(mn, x[i]); mx = fmax(mx, x[i]); }
  }
  group_minmax(mn, mx, lpg);
  double qs = (mx - mn) / (double)levels;
  qs16 = __double2half(qs);
  zp16 = __double2half(mn);
  double qsd = (double)__half2float(qs16), zpd = (double)__half2float(zp16);
  if (active && (!isfinite(qsd) || !isfinite(zpd))) atomicOr(status, 1);
  if (qs > 0.0 && qsd == 0.0) { qs16 = __float2half(5.9604644775390625e-08f); qsd = 5.9604644775390625e-08; }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double c = 0.0;
    if (qsd > 0.0) {
      c = floor((x[i] - zpd) / qsd + 0.5);
      c = fmin(fmax(c, 0.0), (double)levels);
    }
    code[i] = (uint32_t)c;
  }
}


// Fast quantisation of one lane's 4 elements against the reference's float64 grid.
// m32 / err: float32 estimates of the exact float64 values and rigorous bounds on their
// error (|m32 - m| <= err); exact(i) returns the exact float64 value.  The group min / max
// are found exactly from the few candidates whose interval can hold the extreme, and each
// code is decided in float32 unless its rounding interval straddles a grid boundary, in
// which case it is recomputed exactly.  Results are bit-identical to quant4().
template <typename Exact>
__device__ __forceinline__ void quant4_fast(const float (&m32)[4], const float (&err)[4], Exact&& exact,
                                            bool active, int lpg, int levels, uint32_t (&code)[4],
                                            __half& qs16, __half& zp16, int* status) {
  float umin = INFINITY, lmax = -INFINITY;
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { umin = fminf(umin, m32[i] + err[i]); lmax = fmaxf(lmax, m32[i] - err[i]); }
  }
  for (int o = 1; o < lpg; o <<= 1) {
    umin = fminf(umin, __shfl_xor_sync(0xffffffffu, umin, o));
    lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  }
  double mn = INFINITY, mx = -INFINITY;
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool cmin = m32[i] - err[i] <= umin, cmax = m32[i] + err[i] >= lmax;
      if (cmin || cmax) {
        const double e = exact(i);
        if (cmin) mn = fmin(mn, e);
        if (cmax) mx = fmax(mx, e);
      }
    }
  }
  group_minmax(mn, mx, lpg);
  const double qs = (mx - mn) / (double)levels;
  qs16 = __double2half(qs);
  zp16 = __double2half(mn);
  double qsd = (double)__half2float(qs16);
  const double zpd = (double)__half2float(zp16);
  if (active && (!isfinite(qsd) || !isfinite(zpd))) atomicOr(status, 1);
  if (qs > 0.0 && qsd == 0.0) { qs16 = __float2half(5.9604644775390625e-08f); qsd = 5.9604644775390625e-08; }
  const float zpf = (float)zpd, iqs = qsd > 0.0 ? 1.0f / (float)qsd : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t c = 0;
    if (qsd > 0.0) {
      const float t = (m32[i] - zpf) * iqs;
      const float b = (err[i] + fabsf(m32[i] - zpf) * 1.2e-7f) * iqs * 1.0001f + fabsf(t) * 5e-7f + 1e-6f;
      const float lo = fminf(fmaxf(floorf(t + 0.5f - b), 0.f), (float)levels);
      const float hi = fminf(fmaxf(floorf(t + 0.5f + b), 0.f), (float)levels);
      if (lo == hi) {
        c = (uint32_t)lo;
      } else {
        double ce = floor((exact(i) - zpd) / qsd + 0.5);
        c = (uint32_t)fmin(fmax(ce, 0.0), (double)levels);
      }
    }
    code[i] = c;
  }
}

template <int DTY>
__global__ void __launch_bounds__(PACK_WARPS * 32) pack_kernel(PackArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int G = a.D / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y, tile = blockIdx.x;
  double* acc = reinterpret_cast<double*>(smem_raw) + (size_t)warp * G * 64;   // [G][16][4]
  int* cnt = reinterpret_cast<int*>(reinterpret_cast<double*>(smem_raw) + (size_t)PACK_WARPS * G * 64) +
             warp * G * 16;
  for (int i = lane; i < G * 64; i += 32) acc[i] = 0.0;
  for (int i = lane; i < G * 16; i += 32) cnt[i] = 0;
  __syncwarp();

  const int lpg = a.bits > 0 ? a.gs / 4 : 1;
  const int levels = (1 << a.bits) - 1;
  const bool active = lane < G;
  const int c0 = lane * 4;
  constexpr bool FAST = DTY != IN_F64;
  double mu[4], al[4];
  float mu32[4], dmu[4], inva[4];
  bool mule[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mu[i] = active ? a.mu64[(int64_t)u * a.D + c0 + i] : 0.0;
    al[i] = active ? a.alpha64[(int64_t)u * a.D + c0 + i] : 0.0;
    mu32[i] = (float)mu[i];
    mule[i] = mu[i] <= (double)mu32[i];
    dmu[i] = (float)fabs(mu[i] - (double)mu32[i]) * 1.0001f;
    inva[i] = al[i] > 0.0 ? 1.0f / (float)al[i] : 0.f;
  }
  const bool fast = a.signs_fast != nullptr;
  const int64_t tbeg = (int64_t)tile * a.tile, tend = min(a.L, tbeg + a.tile);
  const int rowb = (G + 1) / 2;                    // packed code bytes per token
  const int payb = (a.D * a.bits + 7) / 8;         // payload bytes per token
  const int ngr = a.bits > 0 ? a.D / a.gs : 1;

  for (int64_t t = tbeg + warp; t < tend; t += PACK_WARPS) {
    const int64_t row = ((int64_t)u * a.L + t) * a.D;
    double kp[4];
    uint32_t code = 0;
    uint32_t kc[4] = {0, 0, 0, 0}, vc[4] = {0, 0, 0, 0};
    __half kqs = __float2half(0.f), kzp = kqs, vqs = kqs, vzp = kqs;
    if (FAST) {
      float kf[4] = {0.f, 0.f, 0.f, 0.f}, vf[4] = {0.f, 0.f, 0.f, 0.f};
      if (active) {
        load4<DTY>(a.keys, row + c0, kf);
        load4<DTY>(a.values, row + c0, vf);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        kp[i] = (double)kf[i] - mu[i];
        // K >= mu exactly, decided in float32 (no float32 lies strictly between mu and fl32(mu))
        const bool ge = kf[i] > mu32[i] || (kf[i] == mu32[i] && mule[i]);
        code |= (ge ? 1u : 0u) << (3 - i);
      }
      if (a.codes_in && active)
        code = (a.codes_in[((int64_t)u * a.L + t) * rowb + (lane >> 1)] >> (4 * (lane & 1))) & 15u;
      if (a.bits > 0) {
        float m32[4], e32[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float d = kf[i] - mu32[i];
          if (a.siq) {
            m32[i] = fabsf(d) * inva[i];
            e32[i] = (dmu[i] + fabsf(d) * 2.4e-7f) * inva[i] * 1.0001f + m32[i] * 5e-7f + 1e-37f;
            if (inva[i] == 0.f) { m32[i] = 0.f; e32[i] = 0.f; }
          } else {
            m32[i] = d;
            e32[i] = dmu[i] + fabsf(d) * 1.2e-7f + 1e-37f;
          }
        }
        auto kexact = [&](int i) -> double {
          return a.siq ? (al[i] == 0.0 ? 0.0 : fabs(kp[i]) / al[i]) : kp[i];
        };
        if (a.siq && active) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (m32[i] + e32[i] > 1.0f + 1e-9f && kexact(i) > 1.0 + 1e-9) atomicOr(a.status, 2);
        }
        quant4_fast(m32, e32, kexact, active, lpg, levels, kc, kqs, kzp, a.status);
        const float z4[4] = {0.f, 0.f, 0.f, 0.f};
        quant4_fast(vf, z4, [&](int i) -> double { return (double)vf[i]; }, active, lpg, levels, vc, vqs, vzp,
                    a.status);
      }
    } else {
      double v[4], m[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double k = active ? load_in(a.keys, a.dt, row + c0 + i) : 0.0;
        v[i] = active ? load_in(a.values, a.dt, row + c0 + i) : 0.0;
        kp[i] = k - mu[i];
        code |= (kp[i] >= 0.0 ? 1u : 0u) << (3 - i);
      }
      if (a.codes_in && active)
        code = (a.codes_in[((int64_t)u * a.L + t) * rowb + (lane >> 1)] >> (4 * (lane & 1))) & 15u;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (a.siq) {
          m[i] = al[i] == 0.0 ? 0.0 : fabs(kp[i]) / al[i];
          if (active && m[i] > 1.0 + 1e-9) atomicOr(a.status, 2);
        } else {
          m[i] = kp[i];
        }
      }
      if (a.bits > 0) {   // bits == 0: lossless mode, codes + codebook only
        quant4(m, active, lpg, levels, kc, kqs, kzp, a.status);
        quant4(v, active, lpg, levels, vc, vqs, vzp, a.status);
      }
    }
    // codebook accumulation, token order within this warp's fixed token sequence
    if (active) {
      double* e = acc + ((size_t)lane * 16 + code) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] += kp[i];
      cnt[lane * 16 + code] += 1;
    }

    // -------- reference layout
    uint32_t partner = __shfl_down_sync(0xffffffffu, code, 1);
    if (a.codes_ref && active && !(lane & 1)) {
      uint32_t hi = (lane + 1 < G) ? partner : 0u;
      a.codes_ref[t * rowb + (int64_t)u * a.L * rowb + (lane >> 1)] = (uint8_t)(code | (hi << 4));
    }
    if (a.kq_ref || a.vq_ref) {
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        const uint32_t* cc = which ? vc : kc;
        uint8_t* dst = which ? a.vq_ref : a.kq_ref;
        if (!dst) continue;
        uint8_t* r = dst + ((int64_t)u * a.L + t) * payb;
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) w |= cc[i] << (i * a.bits);
        if (a.bits == 1) {
          uint32_t pw = __shfl_down_sync(0xffffffffu, w, 1);
          if (active && !(lane & 1)) r[lane >> 1] = (uint8_t)(w | ((lane + 1 < G ? pw : 0u) << 4));
        } else if (active) {
          if (a.bits == 2) r[lane] = (uint8_t)w;
          else if (a.bits == 4) { r[2 * lane] = (uint8_t)(w & 0xff); r[2 * lane + 1] = (uint8_t)(w >> 8); }
          else { for (int b = 0; b < 4; ++b) r[4 * lane + b] = (uint8_t)(w >> (8 * b)); }
        }
      }
    }
    if (a.bits > 0 && active && (lane % lpg) == 0) {
      const int64_t pi = ((int64_t)u * a.L + t) * ngr + lane / lpg;
      if (a.ks_ref) { a.ks_ref[pi] = kqs; a.kz_ref[pi] = kzp; }
      if (a.vs_ref) { a.vs_ref[pi] = vqs; a.vz_ref[pi] = vzp; }
    }

    // -------- fast layout (D = 128, bits = 2, gs = 32)
    if (fast) {
      // rotated sign plane: stored byte i = reference byte (t + i) mod 16
      if (!(lane & 1)) {
        int p = lane >> 1;
        int pos = (p - (int)(t & 15)) & 15;
        a.signs_fast[((int64_t)u * a.L + t) * FSIGN + pos] = (uint8_t)(code | (partner << 4));
      }
      if (a.recs_fast) {   // (bits = 0 with only the sign plane: the 16-bit records come from pack16)
      uint32_t out = 0;
      // K4 words 0-15: e2m1 nibbles (sign of K' at bit 3, magnitude code at bits 0-1)
#pragma unroll
      for (int w = 0; w < 16; ++w) {
        uint32_t ck = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int wd, bt;
          k4_pos(c0 + i, wd, bt);
          // sign-in-quant: bit 3 = sign of K'; direct keys: the (unsigned) code alone
          if (wd == w) ck |= (kc[i] | (a.siq && kp[i] < 0.0 ? 8u : 0u)) << bt;
        }
        ck = __reduce_or_sync(0xffffffffu, ck);
        if (lane == w) out = ck;
      }
      // V payload words 16-23
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        uint32_t cv = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int wd, bt;
          vpay_pos(c0 + i, wd, bt);
          if (wd == w) cv |= vc[i] << bt;
        }
        cv = __reduce_or_sync(0xffffffffu, cv);
        if (lane == 16 + w) out = cv;
      }
      // params: group j lives on lanes 8j..8j+7; K params carry 2 qs
      uint32_t kpar = (uint32_t)__half_as_ushort(__hadd(kqs, kqs)) | ((uint32_t)__half_as_ushort(kzp) << 16);
      uint32_t vpar = (uint32_t)__half_as_ushort(vqs) | ((uint32_t)__half_as_ushort(vzp) << 16);
      uint32_t kpj = __shfl_sync(0xffffffffu, kpar, ((lane - 24) & 3) * 8);
      uint32_t vpj = __shfl_sync(0xffffffffu, vpar, ((lane - 28) & 3) * 8);
      if (lane >= 24 && lane < 28) out = kpj;
      if (lane >= 28) out = vpj;
      reinterpret_cast<uint32_t*>(a.recs_fast + ((int64_t)u * a.L + t) * FREC)[lane] = out;
      }
    }
  }
  __syncthreads();
  // fixed-order combine of the warps' partial codebook sums -> this tile's partial
  double* outp = a.cb_part + ((int64_t)u * a.ntiles + tile) * (int64_t)G * 64;
  int* outc = a.cb_cnt + ((int64_t)u * a.ntiles + tile) * (int64_t)G * 16;
  const double* base = reinterpret_cast<const double*>(smem_raw);
  const int* cbase = reinterpret_cast<const int*>(base + (size_t)PACK_WARPS * G * 64);
  for (int i = threadIdx.x; i < G * 64; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < PACK_WARPS; ++w) s += base[(size_t)w * G * 64 + i];
    outp[i] = s;
  }
  for (int i = threadIdx.x; i < G * 16; i += blockDim.x) {
    int s = 0;
    for (int w = 0; w < PACK_WARPS; ++w) s += cbase[w * G * 16 + i];
    outc[i] = s;
  }
}


// ---------------------------------------------------------------- K2': group-parallel quantiser
// D = 128, group 32, bf16 / f32 inputs: one thread per (token, 32-channel group), the 4
// threads of a token are adjacent lanes.  Same arithmetic contract as pack_kernel (float32
// estimates with rigorous error bounds, exact float64 where an estimate is ambiguous), but
// each thread owns a whole quantisation group and builds its share of the fast record in
// registers.  Each CTA loops over a tile of CB_TILE tokens in 64-token blocks and also
// accumulates the tile's codebook partial sums (deterministic order, see the walk below).
//
// Error model (see quant4_fast): every float32 magnitude estimate m_n of channel n satisfies
// |m_n - exact_n| <= e0[n] + |m_n| * 7.5e-7, so the group-wide E = max e0 + max|m| * 7.5e-7
// bounds all of them.  The exact group min (max) can only be attained by channels with
// m_n <= min m + 2E (m_n >= max m - 2E); those few are evaluated in float64.
constexpr int QG_TOK = 64;                 // tokens per 256-thread CTA block
constexpr int CB_TILE = 512;               // tokens per quant_group CTA (one codebook partial each)

__device__ __forceinline__ uint32_t or4(uint32_t v) {   // OR over the 4 lanes of a token
  v |= __shfl_xor_sync(0xffffffffu, v, 1);
  v |= __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// one thread's 32 consecutive input elements, kept packed until they are needed
template <int DTY>
struct Raw32 {
  static constexpr int NW = DTY == IN_BF16 ? 16 : 32;
  uint32_t w[NW];
  __device__ __forceinline__ void load(const void* p, int64_t idx) {
    const uint4* q = DTY == IN_BF16
                         ? reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p) + idx)
                         : reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(p) + idx);
#pragma unroll
    for (int k = 0; k < NW / 4; ++k) {
      const uint4 v = __ldg(q + k);
      w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
    }
  }
  __device__ __forceinline__ float operator[](int n) const {
    if (DTY == IN_BF16) return __uint_as_float((n & 1) ? (w[n >> 1] & 0xFFFF0000u) : (w[n >> 1] << 16));
    return __uint_as_float(w[n]);
  }
};

template <int DTY>
__device__ __forceinline__ float load1(const void* p, int64_t idx) {
  if (DTY == IN_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return reinterpret_cast<const float*>(p)[idx];
}

// packed float32 pairs (sm_100a FFMA2 / FADD2: per lane the same correctly rounded ops)
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

// Quantise one 32-element group (quantizer.py:119-130).  m: float32 estimates, E: group error
// bound (0 = the estimates are exact), [mmin, mmax]: range of m, exact(n): float64 value.
// emit(n, code) ORs a code into the caller's packed words (n is always a compile-time constant);
// reset() clears them; fix[32] is this thread's shared-memory scratch for the exact codes.
// Per-element code decision of the slow path (the fast path's float32 estimate, exact float64
// near rounding boundaries); shared by quant_group32 and the warp-cooperative fix-up below.
struct QgRound {
  float iqs, c0, B;
  double zpd, qsd;
};
template <int BITS>
__device__ __forceinline__ uint32_t qg_code(float m, double exact, const QgRound& r) {
  constexpr int levels = (1 << BITS) - 1;
  constexpr float kRnd = 12582912.f;
  const float x = fmaf(m, r.iqs, r.c0);
  const float y = __fadd_rd(x, kRnd);
  const float fr = x - (y - kRnd);
  if (fr < r.B || fr > 1.f - r.B) {
    const double ce = floor((exact - r.zpd) / r.qsd + 0.5);
    return (uint32_t)fmin(fmax(ce, 0.0), (double)levels);
  }
  return (uint32_t)min(max((int)(__float_as_uint(y) - 0x4B400000u), 0), levels);
}

// Defer: when the whole-group test fails, return true with the rounding parameters in *rp
// (the caller recomputes the group's codes cooperatively) instead of running the per-element
// path on this thread.
template <int BITS, bool Defer = false, typename Exact, typename Emit, typename Reset>
__device__ __forceinline__ bool quant_group32(const float (&m)[32], float E, float mmin, float mmax, Exact&& exact,
                                              Emit&& emit, Reset&& reset, uint8_t* fix, __half& qs16, __half& zp16,
                                              double& mxo, QgRound* rp = nullptr) {
  constexpr int levels = (1 << BITS) - 1;
  double mn, mx;
  if (E == 0.f) {
    mn = (double)mmin;
    mx = (double)mmax;
  } else {
    const float thr_lo = __fadd_ru(mmin, 2.f * E), thr_hi = __fsub_rd(mmax, 2.f * E);
    uint32_t cmin = 0, cmax = 0;
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      cmin |= (m[n] <= thr_lo ? 1u : 0u) << n;
      cmax |= (m[n] >= thr_hi ? 1u : 0u) << n;
    }
    mn = INFINITY;
    mx = -INFINITY;
    for (uint32_t c = cmin | cmax; c; c &= c - 1) {
      const int n = __ffs((int)c) - 1;
      const double e = exact(n);
      if ((cmin >> n) & 1u) mn = fmin(mn, e);
      if ((cmax >> n) & 1u) mx = fmax(mx, e);
    }
  }
  mxo = mx;
  const double qs = (mx - mn) / (double)levels;
  qs16 = __double2half(qs);
  zp16 = __double2half(mn);
  double qsd = (double)__half2float(qs16);
  const double zpd = (double)__half2float(zp16);
  if (qs > 0.0 && qsd == 0.0) { qs16 = __float2half(5.9604644775390625e-08f); qsd = 5.9604644775390625e-08; }
  if (!(qsd > 0.0)) return false;                  // all codes 0
  // x = m * iqs + (0.5 - zp * iqs) estimates T = (exact - zp) / qs + 0.5 with
  // |x - T| <= E iqs (1+2^-23) + |m| iqs 2^-23 + |zp iqs| 2^-22.5 + |x| 2^-24 + 2^-25 < B;
  // codes whose x lies within B of an integer are recomputed exactly afterwards.
  const float zpf = (float)zpd, iqs = 1.0f / (float)qsd;
  const float zq = zpf * iqs, c0 = 0.5f - zq;
  const float mabs = fmaxf(fabsf(mmin), fabsf(mmax)) + E;
  const float B = (E * 1.0001f + mabs * 2.5e-7f) * iqs + fabsf(zq) * 3e-7f + 2e-6f;
  const float omB = 1.f - B;
  constexpr float kRnd = 12582912.f;               // 1.5 * 2^23: x + kRnd (round down) = floor(x)
  // common case, in float32 pairs: every code from its estimate, and one test for the whole
  // group — the largest |frac(x) - 1/2| against 1/2 - B (fr - 1/2 is exact for fr >= 1/4 and
  // off by <= 2^-26 below, hence the 1e-7 margin: anything near a boundary takes the exact path)
  {
    const unsigned long long iq2 = f2pack(iqs, iqs), c02 = f2pack(c0, c0);
    const unsigned long long rnd2 = f2pack(kRnd, kRnd), nrnd2 = f2pack(-kRnd, -kRnd), nh2 = f2pack(-0.5f, -0.5f);
    float amax = 0.f;
#pragma unroll
    for (int n = 0; n < 32; n += 2) {
      unsigned long long x2, y2, t2, r2, d2;
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x2) : "l"(f2pack(m[n], m[n + 1])), "l"(iq2), "l"(c02));
      asm("add.rm.f32x2 %0, %1, %2;" : "=l"(y2) : "l"(x2), "l"(rnd2));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(y2), "l"(nrnd2));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r2) : "l"(x2), "l"(t2));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(r2), "l"(nh2));
      float y0, y1, d0, d1;
      f2unpack(y2, y0, y1);
      f2unpack(d2, d0, d1);
      amax = fmaxf(amax, fmaxf(fabsf(d0), fabsf(d1)));
      const int c0i = min(max((int)(__float_as_uint(y0) - 0x4B400000u), 0), levels);
      const int c1i = min(max((int)(__float_as_uint(y1) - 0x4B400000u), 0), levels);
      emit(n, (uint32_t)c0i);
      emit(n + 1, (uint32_t)c1i);
    }
    if (!(amax > 0.5f - B - 1e-7f)) return false;
    if constexpr (Defer) {
      *rp = QgRound{iqs, c0, B, zpd, qsd};
      return true;
    }
    reset();                                       // rare: redo with per-element decisions
  }
  uint32_t amb = 0;
#pragma unroll
  for (int n = 0; n < 32; ++n) {
    const float x = fmaf(m[n], iqs, c0);
    const float y = __fadd_rd(x, kRnd);
    const float fr = x - (y - kRnd);
    const bool a_n = fr < B || fr > omB;
    int ci = (int)(__float_as_uint(y) - 0x4B400000u);
    ci = min(max(ci, 0), levels);
    amb |= (a_n ? 1u : 0u) << n;
    emit(n, a_n ? 0u : (uint32_t)ci);
  }
  if (amb) {                                       // rare: exact float64 codes via fix[]
    for (uint32_t r = amb; r; r &= r - 1) {
      const int n = __ffs((int)r) - 1;
      const double ce = floor((exact(n) - zpd) / qsd + 0.5);
      fix[n] = (uint8_t)fmin(fmax(ce, 0.0), (double)levels);
    }
#pragma unroll
    for (int n = 0; n < 32; ++n)
      if ((amb >> n) & 1u) emit(n, (uint32_t)fix[n]);
  }
  return false;
}

// Staged K of the 64-token blocks (skewed columns) and their reference code words.  bf16 inputs
// are staged as their own 16-bit words, double-buffered so that the codebook walk over block b
// and the quantisation of block b + 1 need no barrier between them; float32 inputs are staged
// as floats, single-buffered.
template <int DTY>
struct QgSmem {
  static constexpr int NBUF = DTY == IN_BF16 ? 2 : 1;
  using XT = typename std::conditional<DTY == IN_BF16, uint16_t, float>::type;
  XT x[NBUF][QG_TOK][130];
  uint32_t cw[NBUF][QG_TOK][4];
  double acc[4][16][FD];                          // codebook sums per token quarter
  int cnt[16][32];
};
__device__ __forceinline__ float qg_xval(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }
__device__ __forceinline__ float qg_xval(float v) { return v; }

template <int DTY, int BITS>
__global__ void __launch_bounds__(256, 2) quant_group_kernel(PackArgs a) {
  extern __shared__ __align__(16) unsigned char qg_smem[];
  using Smem = QgSmem<DTY>;
  Smem& S = *reinterpret_cast<Smem*>(qg_smem);
  auto& s_x = S.x;
  auto& s_cw = S.cw;
  __shared__ float4 s_c[4][33];                   // (sign threshold, mu32, 1/alpha or 1, -) per channel
  __shared__ double s_mu[4][33], s_al[4][33];
  __shared__ float s_e0max[4];
  __shared__ uint8_t s_fix[256][32];
  const int tid = threadIdx.x, lane = tid & 31, j = tid & 3;
  const int64_t u = blockIdx.y;
  const int tl = tid >> 2;                        // token slot within a 64-token block
  const bool siq = a.siq != 0;
  if (tid < FD) {
    const int c = tid, g = c >> 5, n = c & 31;   // warp g holds group g
    const double mu = a.mu64[u * FD + c], al = a.alpha64[u * FD + c];
    const float m32 = (float)mu;
    const float inva = siq ? (al > 0.0 ? 1.0f / (float)al : 0.f) : 1.f;
    const float dmu = (float)fabs(mu - (double)m32) * 1.0001f;
    const float e0 = (siq ? dmu * inva * 1.0001f : dmu) + 1e-37f;
    // K >= mu  <=>  K >= thr for float32 K (no float32 lies strictly between mu and mu32)
    const float thr = mu <= (double)m32 ? m32 : __int_as_float(__float_as_int(m32) + (m32 >= 0.f ? 1 : -1));
    s_c[g][n] = make_float4(thr, m32, inva, 0.f);
    s_mu[g][n] = mu;
    s_al[g][n] = al;
    const uint32_t emax = __reduce_max_sync(0xffffffffu, __float_as_uint(e0));
    if (n == 0) s_e0max[g] = __uint_as_float(emax);
  }
  for (int q = tid; q < 4 * 16 * FD; q += 256) (&S.acc[0][0][0])[q] = 0.0;
  for (int q = tid; q < 16 * 32; q += 256) (&S.cnt[0][0])[q] = 0;
  // codebook walk: thread (channel pair wp, token quarter wq)
  const int wp = tid & 63, wq = tid >> 6;
  const double wmu0 = a.mu64[u * FD + 2 * wp], wmu1 = a.mu64[u * FD + 2 * wp + 1];
  const int64_t tile0 = (int64_t)blockIdx.x * a.tile, tile1 = min(a.L, tile0 + a.tile);
  __syncthreads();
  auto quant_block = [&](const int64_t b0, const int buf) {
    const int64_t t = b0 + tl;
    const bool valid = t < tile1;
    const int64_t row = (u * a.L + (valid ? t : 0)) * FD + 32 * j;
    Raw32<DTY> kr, vr;
    kr.load(a.keys, row);
    vr.load(a.values, row);
    // sign codes (K >= mu exactly, decided in float32) and key magnitudes
    const uint32_t absmask = siq ? 0x7fffffffu : 0xffffffffu;
    uint32_t geb = 0;                               // bit n: K >= mu for channel 32j + n
    float km[32];
    float kmin = INFINITY, kmax = -INFINITY;
  #pragma unroll
    for (int n = 0; n < 32; ++n) {
      const float4 c = s_c[j][n];
      const float x = kr[n];
      geb |= (x >= c.x ? 1u : 0u) << n;
      km[n] = __uint_as_float(__float_as_uint(x - c.y) & absmask) * c.z;
      kmin = fminf(kmin, km[n]);
      kmax = fmaxf(kmax, km[n]);
    }
    const uint32_t negw = ~geb;
    // cw: word j of the reference code row, channel n at bit 4(n>>2) + 3 - (n&3)
    uint32_t cw = __byte_perm(__brev(geb), 0, 0x0123);
    cw = ((cw >> 4) & 0x0F0F0F0Fu) | ((cw & 0x0F0F0F0Fu) << 4);
    // stage K and the codes for the codebook walk (channel 32j + n at 32j + ((n + 8j) & 31))
    s_cw[buf][tl][j] = cw;
    if constexpr (DTY == IN_BF16) {
      // element pairs (2 n2, 2 n2 + 1) stay adjacent under the skew: one word per pair
      uint32_t* xw = reinterpret_cast<uint32_t*>(&s_x[buf][tl][32 * j]);
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) xw[(n2 + 4 * j) & 15] = kr.w[n2];
    } else {
#pragma unroll
      for (int n = 0; n < 32; ++n) s_x[buf][tl][32 * j + ((n + 8 * j) & 31)] = kr[n];   // 2-way bank conflict at most
    }
    // packed codes: reference words (element n at bit BITS*n of the group's byte string) and,
    // for BITS == 2, this group's share of the fast record words
    constexpr int PER = BITS > 0 ? 32 / BITS : 32;
    uint32_t kref[BITS > 0 ? BITS : 1], vref[BITS > 0 ? BITS : 1];
    uint32_t kp4[4] = {0, 0, 0, 0}, vp8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __half kqs = __float2half(0.f), kzp = kqs, vqs = kqs, vzp = kqs;
    if (BITS > 0) {
  #pragma unroll
      for (int q = 0; q < (BITS > 0 ? BITS : 1); ++q) { kref[q] = 0; vref[q] = 0; }
      {
        const float E = __fmaf_ru(fmaxf(fabsf(kmin), fabsf(kmax)), 7.5e-7f, s_e0max[j]);
        auto kexact = [&](int n) -> double {
          // the K value staged for the codebook walk (the same float; no global reload)
          const double kd = (double)qg_xval(s_x[buf][tl][32 * j + ((n + 8 * j) & 31)]) - s_mu[j][n];
          if (!siq) return kd;
          const double al = s_al[j][n];
          return al == 0.0 ? 0.0 : fabs(kd) / al;
        };
        auto kemit = [&](int n, uint32_t c) {
          kref[n / PER] |= c << (BITS * (n % PER));
          if constexpr (BITS <= 2) {
            // channel 32j + n -> K4 word 4 t4(n) + j, nibble at bit 16(n>>4) + 8e(n) + 4hi(n)
            const int r = n & 15, e = r >> 3, rr = r & 7;
            kp4[rr >> 1] |= c << (16 * (n >> 4) + 8 * e + 4 * (rr & 1));
          }
        };
        auto kreset = [&]() {
#pragma unroll
          for (int q = 0; q < BITS; ++q) kref[q] = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) kp4[q] = 0;
        };
        double kmx;
        quant_group32<BITS>(km, E, kmin, kmax, kexact, kemit, kreset, s_fix[tid], kqs, kzp, kmx);
        if (valid && siq && kmx > 1.0 + 1e-9) atomicOr(a.status, 2);
      }
      {
        float vf[32];
        float vmin = INFINITY, vmax = -INFINITY;
  #pragma unroll
        for (int n = 0; n < 32; ++n) { vf[n] = vr[n]; vmin = fminf(vmin, vf[n]); vmax = fmaxf(vmax, vf[n]); }
        auto vemit = [&](int n, uint32_t c) {
          vref[n / PER] |= c << (BITS * (n % PER));
          if constexpr (BITS <= 2) vp8[n & 7] |= c << (4 * (n >> 4) + 2 * ((n >> 3) & 1));
        };
        auto vreset = [&]() {
#pragma unroll
          for (int q = 0; q < BITS; ++q) vref[q] = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) vp8[q] = 0;
        };
        double vmx;
        QgRound vr2;
        const bool vfail = quant_group32<BITS, true>(vf, 0.f, vmin, vmax, [&](int) -> double { return 0.0; }, vemit,
                                                     vreset, s_fix[tid], vqs, vzp, vmx, &vr2);
        // Groups whose estimates come near a rounding boundary (mostly exact ties of the bf16
        // grid, ~2% of groups) are recomputed by the whole warp, one element per lane, instead
        // of serially by their own thread while the other 31 lanes wait.
        for (uint32_t fm = __ballot_sync(0xffffffffu, vfail); fm; fm &= fm - 1) {
          const int src = __ffs((int)fm) - 1;
          const int64_t srow = __shfl_sync(0xffffffffu, row, src);
          QgRound rr;
          rr.iqs = __shfl_sync(0xffffffffu, vr2.iqs, src);
          rr.c0 = __shfl_sync(0xffffffffu, vr2.c0, src);
          rr.B = __shfl_sync(0xffffffffu, vr2.B, src);
          rr.zpd = __shfl_sync(0xffffffffu, vr2.zpd, src);
          rr.qsd = __shfl_sync(0xffffffffu, vr2.qsd, src);
          const float mv = load1<DTY>(a.values, srow + lane);
          uint8_t* sf = s_fix[(tid & ~31) + src];
          sf[lane] = (uint8_t)qg_code<BITS>(mv, (double)mv, rr);
          __syncwarp();
          if (lane == src) {
            vreset();
            const uint4 c0 = *reinterpret_cast<const uint4*>(sf), c1 = *reinterpret_cast<const uint4*>(sf + 16);
            const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int n = 0; n < 32; ++n) vemit(n, (cw[n >> 2] >> (8 * (n & 3))) & 0xFFu);
          }
          __syncwarp();
        }
      }
      if (valid) {
        const bool kbad = !isfinite(__half2float(kqs)) || !isfinite(__half2float(kzp));
        const bool vbad = !isfinite(__half2float(vqs)) || !isfinite(__half2float(vzp));
        if (kbad || vbad) atomicOr(a.status, 1);
      }
    }
    const int64_t tok = u * a.L + t;
    // ---------------- reference layout
    if (valid && a.codes_ref) reinterpret_cast<uint32_t*>(a.codes_ref + tok * 16)[j] = cw;
    if (valid && BITS > 0) {
      // group j's payload = bytes [4 BITS j, 4 BITS (j + 1)) of the row
      if (a.kq_ref) {
        uint32_t* r = reinterpret_cast<uint32_t*>(a.kq_ref + tok * (16 * BITS) + 4 * BITS * j);
  #pragma unroll
        for (int q = 0; q < BITS; ++q) r[q] = kref[q];
      }
      if (a.vq_ref) {
        uint32_t* r = reinterpret_cast<uint32_t*>(a.vq_ref + tok * (16 * BITS) + 4 * BITS * j);
  #pragma unroll
        for (int q = 0; q < BITS; ++q) r[q] = vref[q];
      }
      const int64_t pi = tok * 4 + j;
      if (a.ks_ref) { a.ks_ref[pi] = kqs; a.kz_ref[pi] = kzp; }
      if (a.vs_ref) { a.vs_ref[pi] = vqs; a.vz_ref[pi] = vzp; }
    }
    // ---------------- fast layout (bits 1 or 2: codes in 2-bit fields; sign-in-quant or direct)
    if constexpr (BITS <= 2) {
      if (a.signs_fast) {
        // rotated sign row: byte i of token t = reference byte (t + i) mod 16
        const int rot = (int)(t & 15), base = lane & ~3;
        const int wsh = rot >> 2, bsh = 8 * (rot & 3);
        const uint32_t lo = __shfl_sync(0xffffffffu, cw, base + ((j + wsh) & 3));
        const uint32_t hi = __shfl_sync(0xffffffffu, cw, base + ((j + wsh + 1) & 3));
        const uint32_t rw = bsh ? ((lo >> bsh) | (hi << (32 - bsh))) : lo;
        // K4 nibbles: bit 3 = sign of K' (1 = negative), bits 0-1 = magnitude code; direct keys
        // keep bit 3 clear (the nibble decodes to code / 2 and zp carries the sign)
        if (siq) {
  #pragma unroll
          for (int n = 0; n < 32; ++n) {
            const int r = n & 15, e = r >> 3, rr = r & 7;
            kp4[rr >> 1] |= ((negw >> n) & 1u) << (16 * (n >> 4) + 8 * e + 4 * (rr & 1) + 3);
          }
        }
        // V payload words g: byte j of every word comes from group j
  #pragma unroll
        for (int q = 0; q < 8; ++q) vp8[q] = or4(vp8[q] << (8 * j));
        // K params carry 2 qs (the e2m1 nibble decodes to sign * code / 2); exact in fp16
        const uint32_t kpar = (uint32_t)__half_as_ushort(__hadd(kqs, kqs)) | ((uint32_t)__half_as_ushort(kzp) << 16);
        const uint32_t vpar = (uint32_t)__half_as_ushort(vqs) | ((uint32_t)__half_as_ushort(vzp) << 16);
        // record words: 0-15 K4 (thread j: words 4 t4 + j), 16-23 V payload (thread j: 16 + 2j,
        // 17 + 2j), 24-27 K params, 28-31 V params
        auto pick8 = [](const uint32_t (&v)[8], int i) {
          uint32_t r = v[0];
  #pragma unroll
          for (int q = 1; q < 8; ++q) r = i == q ? v[q] : r;
          return r;
        };
        if (valid) {
          reinterpret_cast<uint32_t*>(a.signs_fast + tok * FSIGN)[j] = rw;
          uint32_t* rec = reinterpret_cast<uint32_t*>(a.recs_fast + tok * FREC);
  #pragma unroll
          for (int q = 0; q < 4; ++q) rec[4 * q + j] = kp4[q];
          rec[16 + 2 * j] = pick8(vp8, 2 * j);
          rec[17 + 2 * j] = pick8(vp8, 2 * j + 1);
          rec[24 + j] = kpar;
          rec[28 + j] = vpar;
        }
      }
    }
  };
  // codebook walk: thread (channel pair wp, quarter wq) adds K' = fl64(K - mu) of its 16
  // tokens, in token order, to the accumulators of each token's code (codebook.py:128-160)
  auto walk_block = [&](const int64_t b0, const int buf) {
      const int nt = (int)min((int64_t)QG_TOK, tile1 - b0);
      const int jw = wp >> 4, nw = 2 * (wp & 15);
      const int pos = 32 * jw + ((nw + 8 * jw) & 31), sh = 4 * (nw >> 2);
      double2* accw = reinterpret_cast<double2*>(&S.acc[wq][0][2 * wp]);
      int* cntw = &S.cnt[0][wp >> 1];
      const bool counter = (wp & 1) == 0;
      auto step = [&](int i) {
        const uint32_t code = (s_cw[buf][i][jw] >> sh) & 15u;
        float2 x;
        if constexpr (DTY == IN_BF16) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(&s_x[buf][i][pos]);
          x = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
        } else {
          x = *reinterpret_cast<const float2*>(&s_x[buf][i][pos]);
        }
        double2 v = accw[code * (FD / 2)];
        v.x += (double)x.x - wmu0;
        v.y += (double)x.y - wmu1;
        accw[code * (FD / 2)] = v;
        if (counter) atomicAdd(&cntw[code * 32], 1);
      };
      if (nt == QG_TOK) {
#pragma unroll 8
        for (int i = 16 * wq; i < 16 * wq + 16; ++i) step(i);
      } else {
        for (int i = 16 * wq; i < 16 * wq + 16 && i < nt; ++i) step(i);
      }
      };
  constexpr int NB = Smem::NBUF;
  if (tile0 < tile1) quant_block(tile0, 0);
  __syncthreads();
  int buf = 0;
  for (int64_t b0 = tile0; b0 < tile1; b0 += QG_TOK) {
    walk_block(b0, buf);
    const int nbuf = NB == 2 ? buf ^ 1 : 0;
    if constexpr (NB == 1) __syncthreads();        // the next block overwrites the staging
    if (b0 + QG_TOK < tile1) quant_block(b0 + QG_TOK, nbuf);
    __syncthreads();
    buf = nbuf;
  }
  // this tile's partial sums, layout [g][code][i], quarters combined in fixed order
  double* outp = a.cb_part + (u * a.ntiles + blockIdx.x) * (int64_t)(32 * 64);
  int* outc = a.cb_cnt + (u * a.ntiles + blockIdx.x) * (int64_t)(32 * 16);
  for (int q = 0; q < 16; ++q) {
    const int c = tid & (FD - 1);
    if (tid < FD) outp[((c >> 2) * 16 + q) * 4 + (c & 3)] = ((S.acc[0][q][c] + S.acc[1][q][c]) + S.acc[2][q][c]) + S.acc[3][q][c];
  }
  for (int q = tid; q < 32 * 16; q += 256) outc[q] = S.cnt[q & 15][q >> 4];
}

// ---------------------------------------------------------------- K3: codebook finalise
// 256 threads per (unit, 32 consecutive entries): warp w sums tiles w, w + 8, ... in order,
// then the 8 warp sums are combined in warp order (deterministic).
__global__ void __launch_bounds__(256) codebook_final_kernel(int G, int ntiles, const double* __restrict__ part,
                                                             const int* __restrict__ cnt, double* __restrict__ c64,
                                                             float* __restrict__ c32) {
  __shared__ double ws[8][32];
  __shared__ int wn[8][32];
  const int u = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.y * 32 + lane;
  const bool act = i < G * 64;
  double s = 0.0;
  int n = 0;
  if (act) {
    const double* pp = part + (int64_t)u * ntiles * G * 64 + i;
    const int* cp = cnt + (int64_t)u * ntiles * G * 16 + i / 4;
    int t = warp;
    constexpr int UN = 4;
    for (; t + 8 * (UN - 1) < ntiles; t += 8 * UN) {
      double v[UN];
      int c[UN];
#pragma unroll
      for (int k = 0; k < UN; ++k) {
        v[k] = pp[(int64_t)(t + 8 * k) * G * 64];
        c[k] = cp[(int64_t)(t + 8 * k) * G * 16];
      }
#pragma unroll
      for (int k = 0; k < UN; ++k) { s += v[k]; n += c[k]; }
    }
    for (; t < ntiles; t += 8) { s += pp[(int64_t)t * G * 64]; n += cp[(int64_t)t * G * 16]; }
  }
  ws[warp][lane] = s;
  wn[warp][lane] = n;
  __syncthreads();
  if (warp == 0 && act) {
    s = 0.0;
    n = 0;
    for (int w = 0; w < 8; ++w) { s += ws[w][lane]; n += wn[w][lane]; }
    const double c = n > 0 ? s / (double)n : 0.0;
    if (c64) c64[(int64_t)u * G * 64 + i] = c;
    if (c32) c32[(int64_t)u * G * 64 + i] = (float)c;
  }
}

// ---------------------------------------------------------------- full-precision rows
// out_k[u][j][c] = K[u][idx[u][j]][c] - mu[u][c]   (centred, cache.py:269)
// out_v[u][j][c] = V[u][idx[u][j]][c]
template <typename TO>
__global__ void gather_rows_kernel(const void* __restrict__ keys, const void* __restrict__ values,
                                   int dt, int64_t L, int D, const int32_t* __restrict__ idx, int n,
                                   const double* __restrict__ mu64, TO* __restrict__ ok,
                                   TO* __restrict__ ov) {
  const int u = blockIdx.y, j = blockIdx.x;
  const int64_t t = idx[(int64_t)u * n + j];
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    const int64_t src = ((int64_t)u * L + t) * D + c;
    const int64_t dst = ((int64_t)u * n + j) * D + c;
    ok[dst] = (TO)(load_in(keys, dt, src) - mu64[(int64_t)u * D + c]);
    ov[dst] = (TO)load_in(values, dt, src);
  }
}

// decode-time append into the recent ring (cache.py:274-287): one row per unit
template <typename TO>
__global__ void append_kernel(const void* __restrict__ k, const void* __restrict__ v, int dt, int D,
                              const double* __restrict__ mu64, TO* __restrict__ rk, TO* __restrict__ rv,
                              int64_t rcap, int64_t pos, int* __restrict__ status) {
  const int u = blockIdx.x;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double kk = load_in(k, dt, (int64_t)u * D + c), vv = load_in(v, dt, (int64_t)u * D + c);
    if (!isfinite(kk) || !isfinite(vv)) atomicOr(status, 4);
    const int64_t dst = ((int64_t)u * rcap + pos) * D + c;
    rk[dst] = (TO)(kk - mu64[(int64_t)u * D + c]);
    rv[dst] = (TO)vv;
  }
}

// ---------------------------------------------------------------- host launchers
int stats_nsplit(int64_t L) { int64_t n = L / 512; if (n < 1) n = 1; if (n > 64) n = 64; return (int)n; }
constexpr int PACK_TILE = 2048;
// partial-sum tiles: enough for both the generic pack tiles and the codebook tiles
int pack_ntiles(int64_t L) {
  const int64_t a = (L + PACK_TILE - 1) / PACK_TILE, b = (L + CB_TILE - 1) / CB_TILE;
  return (int)(a > b ? a : b);
}

size_t encode_workspace_bytes(int64_t U, int64_t L, int D) {
  size_t a = (size_t)U * stats_nsplit(L) * D * 5 * sizeof(double);
  size_t G = D / 4;
  size_t b = (size_t)U * pack_ntiles(L) * G * 64 * sizeof(double);
  size_t c = (size_t)U * pack_ntiles(L) * G * 16 * sizeof(int);
  return ((a + 255) & ~(size_t)255) + ((b + 255) & ~(size_t)255) + ((c + 255) & ~(size_t)255);
}

cudaError_t launch_encode(const void* keys, const void* values, int dt, int64_t U, int64_t L, int D,
                          int bits, int gs, int siq, int what, const uint8_t* codes_in, double* mu64, double* alpha64, float* mu32,
                          float* alpha32, double* c64, float* c32, uint8_t* codes_ref, uint8_t* kq_ref,
                          __half* ks, __half* kz, uint8_t* vq_ref, __half* vs, __half* vz,
                          uint8_t* signs_fast, uint8_t* recs_fast, void* ws, int* status,
                          cudaStream_t st) {
  const int nsplit = stats_nsplit(L);
  unsigned char* w = reinterpret_cast<unsigned char*>(ws);
  double* spart = reinterpret_cast<double*>(w);
  size_t a = (size_t)U * nsplit * D * 5 * sizeof(double);
  w += (a + 255) & ~(size_t)255;
  const int G = D / 4, ntiles = pack_ntiles(L), ptiles = (int)((L + PACK_TILE - 1) / PACK_TILE);
  double* cbp = reinterpret_cast<double*>(w);
  size_t b = (size_t)U * ntiles * G * 64 * sizeof(double);
  w += (b + 255) & ~(size_t)255;
  int* cbc = reinterpret_cast<int*>(w);

  const int bs = D <= 128 ? 128 : 256;
  if (what & 1) {
    if (dt == IN_BF16 && D % 4 == 0 && D <= 128)
      stats_partial_fast_kernel<IN_BF16><<<dim3((unsigned)U, nsplit), 256, 0, st>>>(keys, L, D, nsplit, spart, status);
    else if (dt == IN_F32 && D % 4 == 0 && D <= 128)
      stats_partial_fast_kernel<IN_F32><<<dim3((unsigned)U, nsplit), 256, 0, st>>>(keys, L, D, nsplit, spart, status);
    else
      stats_partial_kernel<<<dim3((unsigned)U, nsplit), bs, 0, st>>>(keys, dt, L, D, nsplit, spart, status);
    stats_final_kernel<<<dim3((unsigned)U, (D + 7) / 8), 256, 0, st>>>(keys, dt, L, D, nsplit, spart, mu64, alpha64,
                                                                     mu32, alpha32, status);
  }
  if (!(what & 2)) return cudaGetLastError();
  PackArgs pa{keys, values, dt, L, D, bits, gs, siq, mu64, alpha64, codes_ref, kq_ref, ks, kz,
              vq_ref, vs, vz, signs_fast, recs_fast, cbp, cbc, ptiles, PACK_TILE, status, codes_in};
  size_t smem = (size_t)PACK_WARPS * G * 64 * sizeof(double) + (size_t)PACK_WARPS * G * 16 * sizeof(int);
  const bool al16 = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;
  if (D == FD && gs == 32 && (bits == 1 || bits == 2 || bits == 4 || bits == 8) && dt != IN_F64 && !codes_in &&
      al16) {
    const int cnt_tiles = (int)((L + CB_TILE - 1) / CB_TILE);
    if (cnt_tiles > ntiles) return cudaErrorInvalidValue;   // workspace sized by pack_ntiles()
    PackArgs qa = pa;
    qa.tile = CB_TILE;
    qa.ntiles = cnt_tiles;
    const dim3 qg((unsigned)cnt_tiles, (unsigned)U);
    cudaError_t e = cudaSuccess;
    int qsm = 0;
    auto go = [&](auto kern) {
      if (e != cudaSuccess) return;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, qsm);
      if (e == cudaSuccess) kern<<<qg, 256, qsm, st>>>(qa);
    };
    auto run = [&](auto dty) {
      constexpr int DTY = decltype(dty)::value;
      qsm = (int)sizeof(QgSmem<DTY>);
      switch (bits) {
        case 1: go(quant_group_kernel<DTY, 1>); break;
        case 2: go(quant_group_kernel<DTY, 2>); break;
        case 4: go(quant_group_kernel<DTY, 4>); break;
        default: go(quant_group_kernel<DTY, 8>); break;
      }
    };
    if (dt == IN_BF16) run(std::integral_constant<int, IN_BF16>{});
    else run(std::integral_constant<int, IN_F32>{});
    if (e != cudaSuccess) return e;
    codebook_final_kernel<<<dim3((unsigned)U, (G * 64 + 31) / 32), 256, 0, st>>>(G, cnt_tiles, cbp, cbc, c64,
                                                                                  c32);
    return cudaGetLastError();
  }
  auto launch = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(ptiles, (unsigned)U), PACK_WARPS * 32, smem, st>>>(pa);
    return cudaSuccess;
  };
  cudaError_t e = dt == IN_BF16 ? launch(pack_kernel<IN_BF16>) : dt == IN_F32 ? launch(pack_kernel<IN_F32>)
                                                                               : launch(pack_kernel<IN_F64>);
  if (e != cudaSuccess) return e;
  codebook_final_kernel<<<dim3((unsigned)U, (G * 64 + 31) / 32), 256, 0, st>>>(G, ptiles, cbp, cbc, c64, c32);
  return cudaGetLastError();
}

// 16-bit records (the bits = 16 fast path, cache.py:236-238 at model precision): one warp per
// token writes its 128 words: K^ = (K - mu) / alpha-hat (float64, one rounding to fp16) in
// the B-operand order of FREC16 and V in fp16 in the A-operand order.  status bit 4: a V entry
// outside the fp16 range.
__global__ void pack16_kernel(const void* __restrict__ keys, const void* __restrict__ values, int dt, int64_t L,
                              const double* __restrict__ mu64, const float* __restrict__ alpha32,
                              uint8_t* __restrict__ recs16, int* status) {
  const int64_t u = blockIdx.y;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= L) return;
  const int64_t row = (u * L + t) * FD;
  uint32_t* out = reinterpret_cast<uint32_t*>(recs16 + (u * L + t) * FREC16);
  int bad = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int w = lane + 32 * r;
    {   // K word w: chunk t4 = w >> 4, word 2s + e = w & 15 -> channels 16s + 8e + 2t4 (+1)
      const int t4 = w >> 4, s = (w & 15) >> 1, e = w & 1, c = 16 * s + 8 * e + 2 * t4;
      uint32_t h2 = 0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float al = alpha32[u * FD + c + i];
        const double x = (load_in(keys, dt, row + c + i) - mu64[u * FD + c + i]) / (double)(al > 0.f ? al : 1.0f);
        h2 |= (uint32_t)__half_as_ushort(__double2half(x)) << (16 * i);
      }
      out[(k16_off(c) >> 2)] = h2;
    }
    {   // V word w: chunk g = w >> 3, word m = w & 7 -> channels 16m + g (low), 16m + g + 8
      const int g = w >> 3, m = w & 7, c = 16 * m + g;
      const double v0 = load_in(values, dt, row + c), v1 = load_in(values, dt, row + c + 8);
      if (fabs(v0) > 65504.0 || fabs(v1) > 65504.0) bad = 16;
      out[(v16_off(c) >> 2)] = (uint32_t)__half_as_ushort(__double2half(v0)) |
                               ((uint32_t)__half_as_ushort(__double2half(v1)) << 16);
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0 && status) atomicOr(status, bad);
}

cudaError_t launch_pack16(const void* keys, const void* values, int dt, int64_t U, int64_t L, const double* mu64,
                          const float* alpha32, uint8_t* recs16, int* status, cudaStream_t st) {
  if (U == 0 || L == 0) return cudaSuccess;
  pack16_kernel<<<dim3((unsigned)((L + 7) / 8), (unsigned)U), 256, 0, st>>>(keys, values, dt, L, mu64, alpha32,
                                                                            recs16, status);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* keys, const void* values, int dt, int64_t U, int64_t L, int D,
                               const int32_t* idx, int n, const double* mu64, void* ok, void* ov,
                               int out_f64, cudaStream_t st) {
  if (n == 0 || U == 0) return cudaSuccess;
  dim3 grid(n, (unsigned)U);
  if (out_f64)
    gather_rows_kernel<double><<<grid, 128, 0, st>>>(keys, values, dt, L, D, idx, n, mu64,
                                                     (double*)ok, (double*)ov);
  else
    gather_rows_kernel<float><<<grid, 128, 0, st>>>(keys, values, dt, L, D, idx, n, mu64,
                                                    (float*)ok, (float*)ov);
  return cudaGetLastError();
}

cudaError_t launch_append(const void* k, const void* v, int dt, int64_t U, int D, const double* mu64,
                          void* rk, void* rv, int64_t rcap, int64_t pos, int out_f64, int* status,
                          cudaStream_t st) {
  if (out_f64)
    append_kernel<double><<<(unsigned)U, 128, 0, st>>>(k, v, dt, D, mu64, (double*)rk, (double*)rv,
                                                       rcap, pos, status);
  else
    append_kernel<float><<<(unsigned)U, 128, 0, st>>>(k, v, dt, D, mu64, (float*)rk, (float*)rv, rcap,
                                                      pos, status);
  return cudaGetLastError();
}

}  // namespace sikv
