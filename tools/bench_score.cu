// Microbenchmark: pair-table scoring throughput of the sign plane vs warps per SM and
// tokens per batch (no selection, no attention).  Each CTA (one per SM) streams units of
// L tokens (16 B each) from HBM through the same score_batch() the decode kernels use.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_14224_b200/csrc \
//        tools/bench_score.cu -o tools/_bench_score && tools/_bench_score
#include <cstdio>
#include <vector>
#include "decode_common.cuh"

using namespace sikv;

template <int THREADS, int NBX, int CAND, int PF = 1>
__global__ void __launch_bounds__(THREADS, 1)
score_stream(const uint4* __restrict__ signs, int64_t L, int units, float tauf, float* sink, int* cnt) {
  extern __shared__ __align__(16) char T[];
  __shared__ uint32_t segs[THREADS / 32][2 * 512];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 256 * 64; i += THREADS)
    reinterpret_cast<float*>(T)[i] = (float)((i * 2654435761u) >> 20) * 1e-3f;
  __syncthreads();
  const RepKey lb(lane);
  float acc = 0.f;
  int c = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const uint4* p = signs + (int64_t)u * L + tid;
    const int nch = (int)(L / THREADS);
    uint4 wn[PF ? NBX : 1];
    if (PF) {
#pragma unroll
      for (int x = 0; x < NBX; ++x) wn[PF ? x : 0] = __ldg(p + THREADS * x);
    }
    for (int c0 = 0; c0 < nch; c0 += NBX) {
      uint4 w[NBX];
      if (PF) {
#pragma unroll
        for (int x = 0; x < NBX; ++x) w[x] = wn[PF ? x : 0];
        if (c0 + NBX < nch) {
#pragma unroll
          for (int x = 0; x < NBX; ++x) wn[PF ? x : 0] = __ldg(p + (int64_t)THREADS * (c0 + NBX + x));
        }
      } else {
#pragma unroll
        for (int x = 0; x < NBX; ++x) w[x] = __ldg(p + (int64_t)THREADS * (c0 + x));
      }
      float sv[NBX];
      score_batch(w, lb, T, sv);
      if (CAND) {
        uint32_t bits = 0;
#pragma unroll
        for (int x = 0; x < NBX; ++x)
          if (sv[x] >= tauf) bits |= 1u << x;
        const int cn = __popc(bits);
        int inc = cn;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += v;
        }
        int pos = c + inc - cn;
        c += __shfl_sync(0xffffffffu, inc, 31);
        uint32_t* seg = segs[tid >> 5];
        while (bits) {
          const int x = __ffs(bits) - 1;
          bits &= bits - 1;
          float v = sv[0];
#pragma unroll
          for (int y = 1; y < NBX; ++y) v = (x == y) ? sv[y] : v;
          const uint32_t xk = f32_key(v);
          seg[2 * (pos & 511)] = xk;
          seg[2 * (pos & 511) + 1] = (uint32_t)(c0 * THREADS + tid + THREADS * x);
          ++pos;
        }
      } else {
#pragma unroll
        for (int x = 0; x < NBX; ++x) { acc += sv[x]; c += sv[x] >= tauf; }
      }
    }
  }
  sink[blockIdx.x * THREADS + tid] = acc;
  atomicAdd(cnt, c);
}

template <int THREADS, int NBX, int CAND = 0, int PF = 1>
void run(const uint4* d, int64_t L, int units, float* sink, int* cnt, int nsm, float tauf = 1e9f) {
  auto k = score_stream<THREADS, NBX, CAND, PF>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int i = 0; i < 3; ++i) k<<<nsm, THREADS, 65536>>>(d, L, units, tauf, sink, cnt);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 10;
  for (int i = 0; i < it; ++i) k<<<nsm, THREADS, 65536>>>(d, L, units, tauf, sink, cnt);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= it;
  const double bytes = (double)units * L * 16;
  printf("pf %d cand %d threads %4d NB %2d: %.3f ms  %.0f GB/s  (%.0f cycles/unit/SM at 1.965 GHz)\n", PF, CAND, THREADS, NBX, ms,
         bytes / ms / 1e6, ms * 1e-3 * 1.965e9 / ((double)units / nsm));
  (void)PF;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t L = 32768;
  const int units = 4096;
  uint4* d;
  cudaMalloc(&d, (size_t)units * L * 16);
  {
    std::vector<uint32_t> h((size_t)units * L * 4);
    uint32_t x = 12345u;
    for (auto& v : h) { x = x * 1664525u + 1013904223u; v = x; }
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  }
  float* sink;
  int* cnt;
  cudaMalloc(&sink, 1024 * 1024 * 4);
  cudaMalloc(&cnt, 4);
  run<256, 8>(d, L, units, sink, cnt, nsm);
  run<256, 4>(d, L, units, sink, cnt, nsm);
  run<512, 8>(d, L, units, sink, cnt, nsm);
  run<512, 4>(d, L, units, sink, cnt, nsm);
  // tau at ~9% candidates: table entries average 0.5*2^12*1e-3 ~ 2.05 -> score ~ 16 * 2.05
  for (float tau : {36.0f, 38.0f, 40.0f}) {
    cudaMemset(cnt, 0, 4);
    run<256, 8, 1>(d, L, units, sink, cnt, nsm, tau);
    int hc; cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost);
    printf("  tau %.1f: candidate rate %.4f\n", tau, (double)hc / 13.0 / ((double)units * L));
  }
  run<512, 8, 1>(d, L, units, sink, cnt, nsm, 38.0f);
  run<512, 4, 1>(d, L, units, sink, cnt, nsm, 38.0f);
  run<512, 8, 1, 0>(d, L, units, sink, cnt, nsm, 38.0f);
  run<512, 16, 1, 0>(d, L, units, sink, cnt, nsm, 38.0f);
  run<512, 12, 1, 0>(d, L, units, sink, cnt, nsm, 38.0f);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
