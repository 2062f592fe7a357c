// Warp-specialised persistent decode kernel (sm_100a): one 512-thread CTA per SM.
//
//   warps 0-7  (producer, named barrier 1): claim a unit, build its pair table, stream and
//              score its sign plane, collect top-k candidates into a shared-memory slot;
//   warps 8-15 (consumer, named barrier 2): exact k-th key, ordered selection, sparse
//              flash-decode and the output for the unit the producer finished before.
//
// Two slots double-buffer the hand-off (bar.arrive / bar.sync on barriers 3,4 = full and
// 5,6 = empty, 512 threads each), so the HBM stream of unit i+1 overlaps the select +
// attention of unit i.  Units are claimed from a global counter (dynamic balance).  The
// arithmetic is exactly that of decode.cu (shared code in decode_common.cuh).
#include "common.cuh"
#include "select.cuh"
#include "api_types.cuh"
#include "decode_common.cuh"
#include <algorithm>

namespace sikv {

constexpr int WS_THREADS = 512;
__device__ long long* g_prof_ws = nullptr;   // optional per-unit phase clocks (profiling)
__device__ int g_ws_skip = 0;                // debug: bit 0 skips attention, bit 1 skips scoring
using PG = NamedGroup<1, 0>;
using CG = NamedGroup<2, 256>;

template <int ID>
__device__ __forceinline__ void bar_sync512() { asm volatile("bar.sync %0, 512;\n" ::"n"(ID) : "memory"); }
template <int ID>
__device__ __forceinline__ void bar_arrive512() { asm volatile("bar.arrive %0, 512;\n" ::"n"(ID) : "memory"); }
__device__ __forceinline__ void wait_full(int s) { if (s) bar_sync512<4>(); else bar_sync512<3>(); }
__device__ __forceinline__ void arrive_full(int s) { if (s) bar_arrive512<4>(); else bar_arrive512<3>(); }
__device__ __forceinline__ void wait_empty(int s) { if (s) bar_sync512<6>(); else bar_sync512<5>(); }
__device__ __forceinline__ void arrive_empty(int s) { if (s) bar_arrive512<6>(); else bar_arrive512<5>(); }

struct SlotMeta {
  int unit, fb, need_eq, eq_count;
  uint32_t tau, kstar, maxx, pad;
  int wcnt[DW];
};

struct WsArgs {
  const uint8_t* signs;
  const uint8_t* recs;
  const float* cent32;
  const float* alpha32;
  const int32_t* sink_idx;
  const uint32_t* ffrag;
  const float* q;
  float* out;
  float* lse;
  int32_t* sel;
  int32_t* sel_count;
  int32_t* diag;
  int* counter;        // zeroed by the launcher
  uint32_t* gbits;     // [U][2W] fallback bitmaps
  int64_t L, U;
  int fblocks, S, R, Gq, k, capw, sel_stride;
  // shared-memory layout
  int off_pmisc, off_slot, slot_bytes, slot_cand, slot_forced, slot_q, slot_ahat, off_c, c_bits, c_dyn,
      c_stage, off_cmisc;
};

__global__ void __launch_bounds__(WS_THREADS, 1) decode_ws_kernel(WsArgs a) {
  extern __shared__ __align__(128) char sm[];
  const int64_t L = a.L;
  const int W = (int)((L + 31) >> 5);
  const int S = a.S, R = a.R, Gq = a.Gq;

  // role from a value the compiler can prove warp-uniform (keeps uniform-datapath addressing)
  const int role = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 8), 0);
  if (role == 0) {
    // ============================================================ producer
    const int tid = PG::tid();
    char* T = sm;
    float* lut = reinterpret_cast<float*>(sm + a.off_pmisc);
    float* qbar = lut + 512;
    int* th = reinterpret_cast<int*>(qbar + FD);
    uint32_t* tmin = reinterpret_cast<uint32_t*>(th + 256);
    Misc* ms = reinterpret_cast<Misc*>(tmin + 256);
    // per-unit inputs are prefetched into registers one unit ahead (static schedule)
    float pq[4], pal = 0.f;
    float4 pc[2];
    int psid = -1;
    auto prefetch = [&](int64_t u) {
      if (u >= a.U) return;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + DT * i;
        pq[i] = idx < Gq * FD ? a.q[u * Gq * FD + idx] : 0.f;
      }
      pal = tid < FD ? a.alpha32[u * FD + tid] : 0.f;
      const float4* c4 = reinterpret_cast<const float4*>(a.cent32 + u * 32 * 16 * 4);
      pc[0] = c4[tid];
      pc[1] = c4[tid + DT];
      psid = tid < S ? a.sink_idx[u * S + tid] : -1;
    };
    prefetch(blockIdx.x);
    for (int it = 0;; ++it) {
      const int s = it & 1;
      char* slot = sm + a.off_slot + s * a.slot_bytes;
      SlotMeta* meta = reinterpret_cast<SlotMeta*>(slot);
      uint32_t* cand = reinterpret_cast<uint32_t*>(slot + a.slot_cand);
      uint32_t* forced = reinterpret_cast<uint32_t*>(slot + a.slot_forced);
      float* qs = reinterpret_cast<float*>(slot + a.slot_q);
      float* ahat = reinterpret_cast<float*>(slot + a.slot_ahat);
      const int64_t u = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      long long* prof = (g_prof_ws && u < a.U) ? g_prof_ws + u * 12 : nullptr;
      const long long c0 = clock64();
      if (it >= 2) wait_empty(s);
      if (prof && tid == 0) { prof[0] = c0; prof[1] = clock64(); }
      if (u >= a.U) {
        if (tid == 0) meta->unit = -1;
        __threadfence_block();
        arrive_full(s);
        break;
      }
      const uint4* signs = reinterpret_cast<const uint4*>(a.signs + u * L * FSIGN);
      const UnitGeom g = unit_geom(L, S, a.k, a.capw, a.sink_idx + u * S);
      uint4 wsamp[MAX_SAMPLE_CHUNKS];
      load_sample(g, signs, tid, wsamp);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (tid + DT * i < Gq * FD) qs[tid + DT * i] = pq[i];
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
        ahat[tid] = pal > 0.f ? pal : 1.0f;
      }
      PG::sync();
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int e = tid + DT * r, gg = e >> 4;
        const float4 c = pc[r];
        const float q0 = qbar[4 * gg], q1 = qbar[4 * gg + 1], q2 = qbar[4 * gg + 2], q3 = qbar[4 * gg + 3];
        // LUT stored transposed, lutT[code * 32 + group]: the table build below reads it
        // without bank conflicts
        lut[(e & 15) * 32 + gg] = __fadd_rn(__fadd_rn(__fmul_rn(q0, c.x), __fmul_rn(q2, c.z)),
                                            __fadd_rn(__fmul_rn(q1, c.y), __fmul_rn(q3, c.w)));
      }
      PG::sync();
      build_pair_rows<PG>(lut, T);
      if (prof && tid == 0) prof[2] = clock64();
      prefetch(u + gridDim.x);       // next unit's inputs load while this unit streams
      int fb = 0, need_eq = 0, eq_count = 0;
      uint32_t tau = 1, kstar = 0;
      if (g.mode >= 2) {
        fb = produce_candidates<PG>(g, signs, T, forced, wsamp, cand, th, tmin, ms, tau) ? 1 : 0;
        if (fb) {
          uint32_t* gt = a.gbits + u * 2 * W;
          produce_exact<PG>(g, signs, T, forced, reinterpret_cast<int*>(cand), ms, gt, gt + W, kstar, need_eq,
                            eq_count);
        }
      }
      if (prof && tid == 0) prof[3] = clock64();
      if (tid == 0) {
        meta->unit = (int)u;
        meta->fb = fb;
        meta->need_eq = need_eq;
        meta->eq_count = eq_count;
        meta->tau = tau;
        meta->kstar = kstar;
        meta->maxx = ms->maxx;
      }
      if (tid < DW) meta->wcnt[tid] = ms->wcnt[tid];
      __threadfence_block();
      PG::sync();                   // every producer write to the slot and the table use is done
      arrive_full(s);
    }
  } else {
    // ============================================================ consumer
    const int tid = CG::tid(), lane = tid & 31, warp = tid >> 5;
    char* creg = sm + a.off_c;
    int* hist = reinterpret_cast<int*>(creg);
    uint32_t* gt = reinterpret_cast<uint32_t*>(creg + a.c_bits);
    uint32_t* eq = gt + W;
    int32_t* dyn = reinterpret_cast<int32_t*>(creg + a.c_dyn);
    char* stage = creg + a.c_stage + warp * 2 * STAGE_BYTES;
    Misc* ms = reinterpret_cast<Misc*>(sm + a.off_cmisc);
    for (int it = 0;; ++it) {
      const int s = it & 1;
      char* slot = sm + a.off_slot + s * a.slot_bytes;
      const SlotMeta* meta = reinterpret_cast<const SlotMeta*>(slot);
      const uint32_t* cand = reinterpret_cast<const uint32_t*>(slot + a.slot_cand);
      const uint32_t* forced = reinterpret_cast<const uint32_t*>(slot + a.slot_forced);
      const float* qs = reinterpret_cast<const float*>(slot + a.slot_q);
      const float* ahat = reinterpret_cast<const float*>(slot + a.slot_ahat);
      const long long c0 = clock64();
      wait_full(s);
      const int64_t u = meta->unit;
      if (u < 0) break;
      long long* prof = g_prof_ws ? g_prof_ws + u * 12 : nullptr;
      if (prof && tid == 0) { prof[4] = c0; prof[5] = clock64(); }
      const UnitGeom g = unit_geom(L, S, a.k, a.capw, a.sink_idx + u * S);
      const int mode = g.mode;
      uint32_t kstar = meta->kstar;
      int need_eq = meta->need_eq, eq_count = meta->eq_count;
      int32_t* sel_u = a.sel ? a.sel + u * a.sel_stride : nullptr;
      int32_t* sel_count_u = a.sel_count ? a.sel_count + u : nullptr;
      int ndyn;
      if (mode >= 2 && !meta->fb) {
        ndyn = select_emit_candidates<CG>(g, forced, cand, meta->wcnt, meta->maxx, meta->tau, hist, ms, gt, eq, dyn,
                                          sel_u, R, sel_count_u, kstar);
        if (prof && tid == 0) prof[6] = clock64();
      } else {
        if (mode >= 2) {            // the producer's exact path left the bitmaps in global memory
          const uint32_t* src = a.gbits + u * 2 * W;
          for (int i = tid; i < 2 * W; i += DT) (i < W ? gt[i] : eq[i - W]) = __ldcg(src + i);
          CG::sync();
        }
        if (prof && tid == 0) prof[6] = clock64();
        ndyn = emit_selection<CG>(g, mode, forced, gt, eq, need_eq, eq_count, dyn, sel_u, R, sel_count_u, ms);
      }
      if (tid == 0 && a.diag) a.diag[u] = (mode & 3) | (meta->fb ? 4 : 0);
      Attn A;
      attn_init(A, qs, ahat, Gq, lane);
      CG::sync();                   // every consumer read of the slot is done
      arrive_empty(s);
      const int nf = S + R;
      const int nbf = (nf + 15) >> 4;
      if (prof && tid == 0) prof[7] = clock64();
      if (!(g_ws_skip & 1)) {
      attn_forced(A, a.ffrag + u * a.fblocks * 2 * 32 * 32, nf, warp, DW, lane);
      attn_dynamic(A, a.recs + u * L * FREC, dyn, ndyn, (warp - nbf % DW + DW) % DW, DW, stage, lane);
      }
      CG::sync();
      if (prof && tid == 0) prof[8] = clock64();
      float* part = reinterpret_cast<float*>(creg);
      float* pm = part + DW * Gq * FD;
      float* pl = pm + DW * Gq;
      attn_write_partial(A, part, pm, pl, warp, Gq, lane);
      CG::sync();
      attn_merge<CG>(part, pm, pl, DW, Gq, tid, DT, a.out + u * Gq * FD, a.lse ? a.lse + u * Gq : nullptr);
      CG::sync();                   // the region is reused by the next unit
      if (prof && tid == 0) prof[9] = clock64();
    }
  }
}

// ---------------------------------------------------------------- host side
static int a128(int x) { return (x + 127) & ~127; }

struct WsLayout { WsArgs a; int total; };

static WsLayout ws_layout(int64_t L, int k, int S, int Gq, int cap) {
  WsLayout r{};
  WsArgs& a = r.a;
  const int W = (int)((L + 31) / 32);
  const int keff = (int)std::max<int64_t>(0, std::min<int64_t>(k, L - S));
  a.capw = std::max(32, cap / DW);
  int off = TBL_BYTES;
  a.off_pmisc = off;
  off += a128((512 + FD + 256 + 256) * 4 + (int)sizeof(Misc));
  a.off_slot = off;
  int so = a128((int)sizeof(SlotMeta));
  a.slot_cand = so;
  so += a128(std::max(DW * a.capw * 8, (NBIN + 64) * 4));
  a.slot_forced = so;
  so += a128(W * 4);
  a.slot_q = so;
  so += a128(8 * FD * 4);
  a.slot_ahat = so;
  so += a128(FD * 4);
  a.slot_bytes = so;
  off += 2 * so;
  a.off_c = off;
  int co = 0;
  co += a128((NBIN + 64) * 4);
  a.c_bits = co;
  co += a128(2 * W * 4);
  a.c_dyn = co;
  co += a128((std::max(keff, 1) + 16) * 4);
  a.c_stage = co;
  co += DW * 2 * STAGE_BYTES;
  co = std::max(co, a128(DW * Gq * (FD + 2) * 4));
  off += a128(co);
  a.off_cmisc = off;
  off += a128((int)sizeof(Misc));
  r.total = off;
  return r;
}

int ws_smem_bytes(int64_t L, int k, int S, int Gq, int cap) { return ws_layout(L, k, S, Gq, cap).total; }
cudaError_t set_decode_ws_profile(long long* p) { return cudaMemcpyToSymbol(g_prof_ws, &p, sizeof(p)); }
cudaError_t set_decode_ws_skip(int v) { return cudaMemcpyToSymbol(g_ws_skip, &v, sizeof(v)); }
size_t ws_workspace_bytes(int64_t U, int64_t L) { return 256 + (size_t)U * 2 * ((L + 31) / 32) * 4; }

cudaError_t launch_decode_ws(const uint8_t* signs, const uint8_t* recs, const float* cent32, const float* alpha32,
                             const int32_t* sink_idx, int S, const uint32_t* ffrag, int fblocks, int R,
                             const float* q, int64_t U, int64_t L, int Gq, int k, int cap, float* out, float* lse,
                             int32_t* sel, int sel_stride, int32_t* sel_count, int32_t* diag, void* workspace,
                             int nsm, cudaStream_t st) {
  WsLayout lay = ws_layout(L, k, S, Gq, cap);
  WsArgs a = lay.a;
  a.signs = signs; a.recs = recs; a.cent32 = cent32; a.alpha32 = alpha32; a.sink_idx = sink_idx;
  a.ffrag = ffrag; a.q = q; a.out = out; a.lse = lse; a.sel = sel; a.sel_count = sel_count; a.diag = diag;
  a.counter = reinterpret_cast<int*>(workspace);
  a.gbits = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(workspace) + 256);
  a.L = L; a.U = U; a.fblocks = fblocks; a.S = S; a.R = R; a.Gq = Gq; a.k = k; a.sel_stride = sel_stride;
  cudaError_t e = cudaFuncSetAttribute(decode_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(nsm, U);
  decode_ws_kernel<<<grid, WS_THREADS, lay.total, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sikv
