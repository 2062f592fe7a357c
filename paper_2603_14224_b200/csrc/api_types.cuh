// Plain structs shared between the kernels and the C-ABI translation unit.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace sikv {

struct RefPlanes {
  const uint8_t* codes;     // [U][L][ceil(G/2)] packed sign codes
  const uint8_t* kq;        // [U][L][payb]  key magnitudes (siq) or direct keys
  const __half* ks; const __half* kz;   // [U][L][D/gs]
  const uint8_t* vq;
  const __half* vs; const __half* vz;
  const double* kfull; const double* vfull;   // lossless [U][L][D]
  const double* alpha;      // [U][D]
  int bits, gs, siq, D;
  int64_t L;
  // derived (make_planes): bits and group_size are powers of two, so the per-element payload
  // byte / field / group indices are shifts (generic.cu deq_elem)
  int lbits, lper, lgs, payb, ngroups;
};

constexpr int ATT_SPLIT = 16;     // CTAs per (unit, head) of the float64 sparse attention

struct AttendArgs {
  RefPlanes p;
  const double* q;          // [U][H][D]
  int H;
  const int32_t* sel;       // [U][sel_stride]
  const int32_t* nsel;      // [U]
  int sel_stride;
  const int32_t* sink_idx;  // [U][S] sorted
  int S;
  const double* sink_k; const double* sink_v;   // [U][S][D]
  const double* rec_k; const double* rec_v;     // [U][rcap][D]
  int64_t rcap;
  double* ws;               // [U][H][sel_stride]
  double* part;             // [U][H][ATT_SPLIT][130] per-CTA (max, sum, P V) partials
  uint32_t* cnt;            // [U][H] CTAs done
  double* out;              // [U][H][D]
  double* chk;              // [U][H]
};

struct DecodeLayout { int off_cand, off_forced, off_misc, off_bits, off_dyn, off_stage, total, capw; };

}  // namespace sikv
