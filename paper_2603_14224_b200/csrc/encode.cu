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

__global__ void stats_final_kernel(const void* __restrict__ keys, int dt, int64_t L, int D, int nsplit,
                                   const double* __restrict__ part, double* __restrict__ mu64,
                                   double* __restrict__ alpha64, float* __restrict__ mu32,
                                   float* __restrict__ alpha32, int* __restrict__ status) {
  const int u = blockIdx.x;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double sum = -0.0, sab = 0.0, mn = INFINITY, mx = -INFINITY;
    int low = 0x7fffffff;
    for (int s = 0; s < nsplit; ++s) {
      const double* p = part + (((int64_t)u * nsplit + s) * D + c) * 5;
      sum += p[0]; sab += p[1]; mn = fmin(mn, p[2]); mx = fmax(mx, p[3]);
      low = min(low, (int)__double_as_longlong(p[4]));
    }
    bool exact = (low == 0x7fffffff) || (low + 52 < 1023 && sab < ldexp(1.0, low + 52));
    if (!exact) {
      // certificate failed: replay the reference's sequential row order
      atomicOr(status, 8);
      const int64_t base = (int64_t)u * L * D + c;
      sum = load_in(keys, dt, base);
      for (int64_t t = 1; t < L; ++t) sum += load_in(keys, dt, base + t * D);
    }
    double mu = sum / (double)L;
    double a = fmax(fabs(mx - mu), fabs(mn - mu));
    mu64[(int64_t)u * D + c] = mu;
    alpha64[(int64_t)u * D + c] = a;
    if (mu32) mu32[(int64_t)u * D + c] = (float)mu;
    if (alpha32) alpha32[(int64_t)u * D + c] = (float)a;
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
  double mu[4], al[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mu[i] = active ? a.mu64[(int64_t)u * a.D + c0 + i] : 0.0;
    al[i] = active ? a.alpha64[(int64_t)u * a.D + c0 + i] : 0.0;
  }
  const bool fast = a.signs_fast != nullptr;
  const int64_t tbeg = (int64_t)tile * a.tile, tend = min(a.L, tbeg + a.tile);
  const int rowb = (G + 1) / 2;                    // packed code bytes per token
  const int payb = (a.D * a.bits + 7) / 8;         // payload bytes per token
  const int ngr = a.bits > 0 ? a.D / a.gs : 1;

  for (int64_t t = tbeg + warp; t < tend; t += PACK_WARPS) {
    const int64_t row = ((int64_t)u * a.L + t) * a.D;
    double kp[4], v[4], m[4];
    uint32_t code = 0;
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
    // codebook accumulation, token order within this warp's fixed token sequence
    if (active) {
      double* e = acc + ((size_t)lane * 16 + code) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] += kp[i];
      cnt[lane * 16 + code] += 1;
    }
    uint32_t kc[4] = {0, 0, 0, 0}, vc[4] = {0, 0, 0, 0};
    __half kqs = __float2half(0.f), kzp = kqs, vqs = kqs, vzp = kqs;
    if (a.bits > 0) {   // bits == 0: lossless mode, codes + codebook only
      quant4(m, active, lpg, levels, kc, kqs, kzp, a.status);
      quant4(v, active, lpg, levels, vc, vqs, vzp, a.status);
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
      uint32_t out = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        uint32_t ck = 0, cv = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int wd, bt;
          kpay_pos(c0 + i, wd, bt);
          if (wd == w) ck |= kc[i] << bt;
          vpay_pos(c0 + i, wd, bt);
          if (wd == w) cv |= vc[i] << bt;
        }
        ck = __reduce_or_sync(0xffffffffu, ck);
        cv = __reduce_or_sync(0xffffffffu, cv);
        if (lane == w) out = ck;
        if (lane == 8 + w) out = cv;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t sg = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int wd, bt;
          ksgn_pos(c0 + i, wd, bt);
          if (wd == w && kp[i] < 0.0) sg |= 1u << bt;   // 1 = negative
        }
        sg = __reduce_or_sync(0xffffffffu, sg);
        if (lane == 24 + w) out = sg;
      }
      // params: group j lives on lanes 8j..8j+7
      uint32_t kpar = (uint32_t)__half_as_ushort(kqs) | ((uint32_t)__half_as_ushort(kzp) << 16);
      uint32_t vpar = (uint32_t)__half_as_ushort(vqs) | ((uint32_t)__half_as_ushort(vzp) << 16);
      uint32_t kpj = __shfl_sync(0xffffffffu, kpar, ((lane - 16) & 3) * 8);
      uint32_t vpj = __shfl_sync(0xffffffffu, vpar, ((lane - 20) & 3) * 8);
      if (lane >= 16 && lane < 20) out = kpj;
      if (lane >= 20 && lane < 24) out = vpj;
      if (lane >= 28) out = 0;
      reinterpret_cast<uint32_t*>(a.recs_fast + ((int64_t)u * a.L + t) * FREC)[lane] = out;
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

// ---------------------------------------------------------------- K3: codebook finalise
__global__ void codebook_final_kernel(int G, int ntiles, const double* __restrict__ part,
                                      const int* __restrict__ cnt, double* __restrict__ c64,
                                      float* __restrict__ c32) {
  const int u = blockIdx.x;
  for (int i = threadIdx.x; i < G * 64; i += blockDim.x) {
    double s = 0.0;
    int n = 0;
    for (int t = 0; t < ntiles; ++t) {
      s += part[((int64_t)u * ntiles + t) * G * 64 + i];
      n += cnt[((int64_t)u * ntiles + t) * G * 16 + i / 4];
    }
    double c = n > 0 ? s / (double)n : 0.0;
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
constexpr int PACK_TILE = 512;
int pack_ntiles(int64_t L) { return (int)((L + PACK_TILE - 1) / PACK_TILE); }

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
  const int G = D / 4, ntiles = pack_ntiles(L);
  double* cbp = reinterpret_cast<double*>(w);
  size_t b = (size_t)U * ntiles * G * 64 * sizeof(double);
  w += (b + 255) & ~(size_t)255;
  int* cbc = reinterpret_cast<int*>(w);

  const int bs = D <= 128 ? 128 : 256;
  if (what & 1) {
    stats_partial_kernel<<<dim3((unsigned)U, nsplit), bs, 0, st>>>(keys, dt, L, D, nsplit, spart, status);
    stats_final_kernel<<<(unsigned)U, bs, 0, st>>>(keys, dt, L, D, nsplit, spart, mu64, alpha64, mu32,
                                                   alpha32, status);
  }
  if (!(what & 2)) return cudaGetLastError();
  PackArgs pa{keys, values, dt, L, D, bits, gs, siq, mu64, alpha64, codes_ref, kq_ref, ks, kz,
              vq_ref, vs, vz, signs_fast, recs_fast, cbp, cbc, ntiles, PACK_TILE, status, codes_in};
  size_t smem = (size_t)PACK_WARPS * G * 64 * sizeof(double) + (size_t)PACK_WARPS * G * 16 * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  pack_kernel<<<dim3(ntiles, (unsigned)U), PACK_WARPS * 32, smem, st>>>(pa);
  codebook_final_kernel<<<(unsigned)U, 256, 0, st>>>(G, ntiles, cbp, cbc, c64, c32);
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
