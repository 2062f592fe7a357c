// extern "C" boundary of libsikv_b200.so: argument validation, error reporting, launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <string>
#include <cstring>
#include <algorithm>

#include "../../include/sikv_b200.h"
#include "common.cuh"
#include "api_types.cuh"

namespace sikv {
// encode.cu
size_t encode_workspace_bytes(int64_t U, int64_t L, int D);
cudaError_t launch_encode(const void*, const void*, int, int64_t, int64_t, int, int, int, int, int,
                          const uint8_t*, double*, double*, float*, float*, double*, float*, uint8_t*,
                          uint8_t*, __half*, __half*, uint8_t*, __half*, __half*, uint8_t*, uint8_t*, void*,
                          int*, cudaStream_t);
cudaError_t launch_pack16(const void*, const void*, int, int64_t, int64_t, const double*, const float*, uint8_t*, int*,
                          cudaStream_t);
cudaError_t launch_gather_rows(const void*, const void*, int, int64_t, int64_t, int, const int32_t*, int,
                               const double*, void*, void*, int, cudaStream_t);
cudaError_t launch_append(const void*, const void*, int, int64_t, int, const double*, void*, void*, int64_t,
                          int64_t, int, int*, cudaStream_t);
// decode.cu
DecodeLayout decode_layout(int64_t L, int k, int S, int Gq, int cap);
cudaError_t launch_decode(const uint8_t*, const uint8_t*, const float*, const float*, const int32_t*, int,
                          const uint32_t*, int, const int32_t*, int, const float*, int64_t, int64_t, int, int, int, float*,
                          float*, int32_t*, int, int32_t*, int32_t*, const int32_t*, int, cudaStream_t, int*);
cudaError_t launch_pack_forced(const float*, const float*, int, const float*, const float*, int64_t, const int32_t*,
                               int, const float*, int64_t, int, int, int, uint32_t*, int*, cudaStream_t);
cudaError_t launch_append_forced(const void*, const void*, int, int64_t, const int32_t*, const double*, const float*,
                                 const float*, const float*, int, float*, float*, int64_t, int32_t*, int, uint32_t*,
                                 int*, cudaStream_t);
cudaError_t launch_score_fast(const uint8_t*, const float*, const float*, int, int64_t, int64_t, int, float*,
                              cudaStream_t);
cudaError_t set_decode_profile(long long*);
cudaError_t set_k1_skip(int);
cudaError_t set_decode_two_profile(long long*);
cudaError_t set_decode_split_profile(long long*);
int split_smem_bytes(int64_t L, int k, int S, int Gq, int cap, int ns);
int split_default_cap(int64_t L, int k, int S, int ns);
cudaError_t launch_decode_split(const uint8_t*, const uint8_t*, const float*, const float*, const int32_t*, int,
                                const uint32_t*, int, const int32_t*, int, const float*, int64_t, int64_t, int, int, int, int, float*,
                                float*, int32_t*, int, int32_t*, int32_t*, const int32_t*, int, cudaStream_t);
int two_select_smem_bytes(int64_t L, int k, int S, int cap, int Gq);
int two_attend_smem_bytes(int64_t L, int k, int S, int Gq, bool rec16);
size_t two_workspace_bytes(int64_t U, int64_t L, int k, int S);
cudaError_t launch_decode_two(const uint8_t*, const uint8_t*, const float*, const float*, const int32_t*, int,
                              const uint32_t*, int, const int32_t*, int, const float*, int64_t, int64_t, int, int, int, float*, float*,
                              int32_t*, int, int32_t*, int32_t*, void*, int, const int32_t*, int, const sikv_exchange*,
                              cudaStream_t);
cudaError_t launch_push_outputs(const sikv_exchange& x, const float* out, int64_t U, int Gq, cudaStream_t st);
cudaError_t launch_exchange_wait(const unsigned long long* flag, unsigned long long target, cudaStream_t st);
// snapkv.cu
size_t snap_workspace_bytes(int64_t U, int64_t L, int w);
cudaError_t launch_snap_pooled(const void*, int, int64_t, int64_t, int, const double*, const double*, int, int, void*,
                               double**, cudaStream_t);
// generic.cu
cudaError_t launch_lut_f64(const double*, const double*, int64_t, int, int, double*, cudaStream_t);
cudaError_t launch_score_f64(const double*, const uint8_t*, int64_t, int, int64_t, double*, cudaStream_t);
size_t topk_workspace_bytes(int64_t U, int64_t L);
cudaError_t launch_topk(const void*, int, int64_t, int64_t, const int32_t*, int, int, void*, int32_t*, int,
                        int32_t*, cudaStream_t);
cudaError_t launch_dequant_rows(const RefPlanes&, int64_t, const int64_t*, int64_t, int, double*, cudaStream_t);
cudaError_t launch_attend_f64(const AttendArgs&, int64_t, cudaStream_t);
cudaError_t launch_center(const void*, int, int64_t, int64_t, int, const double*, double*, cudaStream_t);
}  // namespace sikv

using namespace sikv;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_ret(cudaError_t e, const char* where) {
  if (e == cudaSuccess) { g_err.clear(); return SIKV_OK; }
  return fail(SIKV_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define REQUIRE(cond, code, msg) \
  do { if (!(cond)) return fail((code), (msg)); } while (0)

static bool good_dtype(int d) { return d == IN_F32 || d == IN_F64 || d == IN_BF16; }
static bool good_bits(int b) { return b == 1 || b == 2 || b == 4 || b == 8; }
static bool good_group(int g) { return g == 4 || g == 8 || g == 16 || g == 32 || g == 64 || g == 128; }
static int num_sms() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}
// The first runtime call of this library binds the calling thread's current context.  When
// that first call is a kernel launch the runtime probes an invalid kernel handle once (a
// reported API error under compute-sanitizer), so every launching entry point binds first.
static void rt_bind() {
  static thread_local bool bound = false;
  if (bound) return;
  cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;   // legal while a capture is active
  cudaThreadExchangeStreamCaptureMode(&m);
  cudaFree(nullptr);
  cudaThreadExchangeStreamCaptureMode(&m);
  bound = true;
}
static int max_smem() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

extern "C" {

const char* sikv_last_error(void) { return g_err.c_str(); }
int sikv_abi_version(void) { return 8; }

size_t sikv_encode_workspace_bytes(int64_t units, int64_t tokens, int64_t dim) {
  return encode_workspace_bytes(units, tokens, (int)dim);
}

int sikv_encode(const void* keys, const void* values, int in_dtype, int64_t units, int64_t tokens,
                int64_t dim, int bits, int group_size, int sign_in_quant, int what,
                const uint8_t* codes_in, double* mu64, double* alpha64, float* mu32, float* alpha32,
                double* cent64, float* cent32, uint8_t* codes_ref, uint8_t* kq_ref,
                uint16_t* kq_scales, uint16_t* kq_zeros, uint8_t* vq_ref, uint16_t* vq_scales,
                uint16_t* vq_zeros, uint8_t* signs_fast, uint8_t* recs_fast, void* workspace,
                size_t workspace_bytes, int* status_dev, void* stream) {
  rt_bind();
  REQUIRE(keys && values && mu64 && alpha64 && status_dev, SIKV_EINVAL, "null required pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "in_dtype must be 0 (f32), 1 (f64) or 2 (bf16)");
  REQUIRE(units >= 1 && tokens >= 1, SIKV_EINVAL, "keys must contain at least one row");
  REQUIRE(dim >= 1, SIKV_EINVAL, "channel count must be positive");
  if (what & 2) {
    REQUIRE(dim >= 4 && dim % 4 == 0, SIKV_EINVAL, "channel count must be a positive multiple of 4");
    REQUIRE(dim <= 128, SIKV_EUNSUPPORTED, "encoder supports dim <= 128");
  }
  REQUIRE(bits == 0 || good_bits(bits), SIKV_EINVAL, "bits must be one of (1, 2, 4, 8) or 0 (lossless)");
  REQUIRE(!(what & 2) || bits == 0 || (good_group(group_size) && dim % group_size == 0), SIKV_EINVAL,
          "channel count not divisible by group_size (group_size must be 4..128, power of two)");
  REQUIRE(what >= 1 && what <= 3, SIKV_EINVAL, "what must be 1, 2 or 3");
  if (what & 2) {
    REQUIRE(cent64 || cent32, SIKV_EINVAL, "pack needs a centroid output");
    REQUIRE(workspace && workspace_bytes >= encode_workspace_bytes(units, tokens, (int)dim), SIKV_EINVAL,
            "workspace too small (sikv_encode_workspace_bytes)");
  } else {
    REQUIRE(workspace && workspace_bytes >= encode_workspace_bytes(units, tokens, (int)dim), SIKV_EINVAL,
            "workspace too small (sikv_encode_workspace_bytes)");
  }
  if (signs_fast || recs_fast) {
    REQUIRE(signs_fast && (recs_fast || bits == 0), SIKV_EINVAL,
            "fast layout needs both signs_fast and recs_fast (bits 0: signs_fast alone, for 16-bit records)");
    REQUIRE(dim == 128 && (bits == 1 || bits == 2 || (bits == 0 && !recs_fast)) && group_size == 32,
            SIKV_EUNSUPPORTED, "fast layout requires dim=128, bits 1 or 2 (0: sign plane only), group_size=32");
  }
  if (kq_ref) REQUIRE(kq_scales && kq_zeros, SIKV_EINVAL, "kq_ref needs scales and zeros");
  if (vq_ref) REQUIRE(vq_scales && vq_zeros, SIKV_EINVAL, "vq_ref needs scales and zeros");
  cudaError_t e = launch_encode(keys, values, in_dtype, units, tokens, (int)dim, bits, group_size,
                                sign_in_quant, what, codes_in, mu64, alpha64, mu32, alpha32, cent64, cent32,
                                codes_ref, kq_ref, (__half*)kq_scales, (__half*)kq_zeros, vq_ref,
                                (__half*)vq_scales, (__half*)vq_zeros, signs_fast, recs_fast, workspace,
                                status_dev, (cudaStream_t)stream);
  return cuda_ret(e, "sikv_encode");
}

int sikv_gather_rows(const void* keys, const void* values, int in_dtype, int64_t units, int64_t tokens,
                     int64_t dim, const int32_t* idx, int64_t n, const double* mu64, void* out_k, void* out_v,
                     int out_f64, void* stream) {
  rt_bind();
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "bad in_dtype");
  REQUIRE(n >= 0 && units >= 1 && tokens >= 1 && dim >= 1, SIKV_EINVAL, "bad shape");
  if (n == 0) return SIKV_OK;
  REQUIRE(keys && values && idx && mu64 && out_k && out_v, SIKV_EINVAL, "null pointer");
  return cuda_ret(launch_gather_rows(keys, values, in_dtype, units, tokens, (int)dim, idx, (int)n, mu64, out_k,
                                     out_v, out_f64, (cudaStream_t)stream),
                  "sikv_gather_rows");
}

int sikv_append(const void* k, const void* v, int in_dtype, int64_t units, int64_t dim, const double* mu64,
                void* recent_k, void* recent_v, int64_t rcap, int64_t pos, int out_f64, int* status_dev,
                void* stream) {
  rt_bind();
  REQUIRE(k && v && mu64 && recent_k && recent_v && status_dev, SIKV_EINVAL, "null pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "bad in_dtype");
  REQUIRE(pos >= 0 && pos < rcap, SIKV_EINVAL, "recent buffer full (pos >= rcap)");
  return cuda_ret(launch_append(k, v, in_dtype, units, (int)dim, mu64, recent_k, recent_v, rcap, pos, out_f64,
                                status_dev, (cudaStream_t)stream),
                  "sikv_append");
}

int sikv_decode_default_cap(int64_t tokens, int k, int sinks) {
  // Candidate buffer: ~2k + 1024 entries (the sampled threshold keeps ~k + 4 sqrt(k') of them),
  // shrunk (not below ~1.4k + 512) only when that lets two CTAs share an SM (2 x 113 KB).
  const int64_t ncand = std::max<int64_t>(tokens - sinks, 0);
  const int64_t keff = std::min<int64_t>(k, ncand);
  if (keff == 0 || keff == ncand) return 1024;        // no candidate selection needed
  int64_t cap = std::max<int64_t>(2 * keff + 1024, 1024);
  const int64_t floor_cap = std::max<int64_t>(keff + keff * 2 / 5 + 512, 1024);
  if (decode_layout(tokens, k, sinks, 8, (int)floor_cap).total > 113 * 1024) return (int)cap;
  while (cap > floor_cap && decode_layout(tokens, k, sinks, 8, (int)cap).total > 113 * 1024) cap -= 64;
  return (int)cap;
}

int sikv_decode_smem_bytes(int64_t tokens, int k, int sinks, int gq, int cap) {
  if (cap <= 0) cap = sikv_decode_default_cap(tokens, k, sinks);
  return decode_layout(tokens, k, sinks, gq, cap).total;
}

int sikv_pack16(const void* keys, const void* values, int in_dtype, int64_t units, int64_t tokens,
                const double* mu64, const float* alpha32, uint8_t* recs16, int* status_dev, void* stream) {
  rt_bind();
  REQUIRE(keys && values && mu64 && alpha32 && recs16, SIKV_EINVAL, "null pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "in_dtype must be 0 (f32), 1 (f64) or 2 (bf16)");
  REQUIRE(units >= 0 && tokens >= 0, SIKV_EINVAL, "bad shape");
  return cuda_ret(launch_pack16(keys, values, in_dtype, units, tokens, mu64, alpha32, recs16, status_dev,
                                (cudaStream_t)stream),
                  "sikv_pack16");
}

int sikv_forced_blocks(int sinks, int64_t rcap) { return (int)std::max<int64_t>(1, (sinks + rcap + 15) / 16); }

int sikv_forced_block_words(void) { return FBLK_WORDS; }

int sikv_pack_forced(const float* sink_k, const float* sink_v, int sinks, const float* recent_k,
                     const float* recent_v, int64_t rcap, const int32_t* recent_n, int recent, const float* alpha32,
                     int64_t units, uint32_t* forced_frag, int frag_blocks, int row_begin, int row_end,
                     int* status_dev, void* stream) {
  rt_bind();
  REQUIRE(alpha32 && forced_frag, SIKV_EINVAL, "null pointer");
  REQUIRE(sinks == 0 || (sink_k && sink_v), SIKV_EINVAL, "sink rows missing");
  REQUIRE(rcap == 0 || (recent_k && recent_v), SIKV_EINVAL, "recent rows missing");
  REQUIRE(recent >= 0 && recent <= rcap, SIKV_EINVAL, "recent count out of range");
  REQUIRE(frag_blocks >= sikv_forced_blocks(sinks, rcap), SIKV_EINVAL, "frag_blocks too small");
  REQUIRE(row_begin >= 0 && row_end >= row_begin, SIKV_EINVAL, "bad row range");
  const int b0 = row_begin / 16, b1 = std::min(frag_blocks, (row_end + 15) / 16);
  return cuda_ret(launch_pack_forced(sink_k, sink_v, sinks, recent_k, recent_v, rcap, recent_n, recent, alpha32,
                                     units, frag_blocks, b0, b1, forced_frag, status_dev, (cudaStream_t)stream),
                  "sikv_pack_forced");
}

int sikv_append_forced(const void* k, const void* v, int in_dtype, int64_t n, const int32_t* unit_ids,
                       const double* mu64, const float* alpha32, const float* sink_k, const float* sink_v, int sinks,
                       float* recent_k, float* recent_v, int64_t rcap, int32_t* recent_n, uint32_t* forced_frag,
                       int frag_blocks, int* status_dev, void* stream) {
  rt_bind();
  REQUIRE(k && v && mu64 && alpha32 && recent_k && recent_v && recent_n && forced_frag, SIKV_EINVAL, "null pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "in_dtype must be 0 (f32), 1 (f64) or 2 (bf16)");
  REQUIRE(n >= 0 && rcap >= 1, SIKV_EINVAL, "bad row count or capacity");
  REQUIRE(sinks == 0 || (sink_k && sink_v), SIKV_EINVAL, "sink rows missing");
  REQUIRE(frag_blocks >= sikv_forced_blocks(sinks, rcap), SIKV_EINVAL, "frag_blocks too small");
  return cuda_ret(launch_append_forced(k, v, in_dtype, n, unit_ids, mu64, alpha32, sink_k, sink_v, sinks, recent_k,
                                       recent_v, rcap, recent_n, frag_blocks, forced_frag, status_dev,
                                       (cudaStream_t)stream),
                  "sikv_append_forced");
}

size_t sikv_decode_workspace_bytes(int64_t units, int64_t tokens) {
  return two_workspace_bytes(units, tokens, (int)std::min<int64_t>(tokens, 1 << 30), 0);
}
size_t sikv_decode_workspace_bytes_k(int64_t units, int64_t tokens, int k, int sinks) {
  return two_workspace_bytes(units, tokens, k, sinks);
}

static thread_local int g_last_decode_kernel = 0;
int sikv_decode_last_kernel() { return g_last_decode_kernel; }

int sikv_decode_step(const uint8_t* signs_fast, const uint8_t* recs_fast, const float* cent32,
                     const float* alpha32, const int32_t* sink_idx, int sinks, const uint32_t* forced_frag,
                     int frag_blocks, const int32_t* recent_n, int recent, const float* q, int64_t units,
                     int64_t tokens, int gq, int k,
                     int cap, float* out, float* lse, int32_t* sel, int sel_stride, int32_t* sel_count,
                     int32_t* diag, void* workspace, size_t workspace_bytes, const int32_t* unit_map,
                     int lut_mode, int kernel, void* stream) {
  return sikv_decode_step_x(signs_fast, recs_fast, cent32, alpha32, sink_idx, sinks, forced_frag, frag_blocks,
                            recent_n, recent, q, units, tokens, gq, k, cap, out, lse, sel, sel_stride, sel_count,
                            diag, workspace, workspace_bytes, unit_map, lut_mode, kernel, nullptr, stream);
}

static int check_exchange(const sikv_exchange* x) {
  REQUIRE(x->npeers >= 0 && x->npeers <= SIKV_MAX_PEERS, SIKV_EINVAL, "npeers must be 0..8");
  if (x->npeers == 0) return SIKV_OK;
  REQUIRE(x->unit_gid, SIKV_EINVAL, "the exchange needs unit_gid");
  for (int p = 0; p < x->npeers; ++p)
    REQUIRE(x->out[p] && x->flag[p], SIKV_EINVAL, "null peer buffer or counter");
  return SIKV_OK;
}

int sikv_exchange_wait(const unsigned long long* flag, unsigned long long target, void* stream) {
  rt_bind();
  REQUIRE(flag, SIKV_EINVAL, "null counter");
  return cuda_ret(launch_exchange_wait(flag, target, (cudaStream_t)stream), "sikv_exchange_wait");
}

int sikv_ipc_handle(const void* dev_ptr, void* handle64, size_t* offset) {
  rt_bind();
  REQUIRE(dev_ptr && handle64 && offset, SIKV_EINVAL, "null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // the handle names the whole allocation (a caching allocator hands out interior pointers):
  // its base from the driver (entry point looked up at run time, no libcuda link)
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(SIKV_ECUDA, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  REQUIRE(get_range(&base, &size, (CUdeviceptr)dev_ptr) == CUDA_SUCCESS, SIKV_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e == cudaSuccess) {
    memcpy(handle64, &h, sizeof(h));
    *offset = (size_t)((CUdeviceptr)dev_ptr - base);
  }
  return cuda_ret(e, "sikv_ipc_handle");
}

int sikv_ipc_open(const void* handle64, void** dev_ptr) {
  rt_bind();
  REQUIRE(handle64 && dev_ptr, SIKV_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return cuda_ret(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "sikv_ipc_open");
}

int sikv_ipc_close(void* dev_ptr) {
  rt_bind();
  REQUIRE(dev_ptr, SIKV_EINVAL, "null pointer");
  return cuda_ret(cudaIpcCloseMemHandle(dev_ptr), "sikv_ipc_close");
}

int sikv_decode_step_x(const uint8_t* signs_fast, const uint8_t* recs_fast, const float* cent32,
                       const float* alpha32, const int32_t* sink_idx, int sinks, const uint32_t* forced_frag,
                       int frag_blocks, const int32_t* recent_n, int recent, const float* q, int64_t units,
                       int64_t tokens, int gq, int k,
                       int cap, float* out, float* lse, int32_t* sel, int sel_stride, int32_t* sel_count,
                       int32_t* diag, void* workspace, size_t workspace_bytes, const int32_t* unit_map,
                       int lut_mode, int kernel, const sikv_exchange* xchg, void* stream) {
  rt_bind();
  if (xchg) {
    const int rc = check_exchange(xchg);
    if (rc != SIKV_OK) return rc;
    if (xchg->npeers == 0) xchg = nullptr;
  }
  // paths without the fused epilogue push after their kernel, on the same stream
  auto push = [&](cudaError_t e) -> cudaError_t {
    if (e != cudaSuccess || !xchg) return e;
    return launch_push_outputs(*xchg, out, units, gq, (cudaStream_t)stream);
  };
  REQUIRE(signs_fast && recs_fast && cent32 && alpha32 && q && out, SIKV_EINVAL, "null required pointer");
  REQUIRE(units >= 1 && tokens >= 1, SIKV_EINVAL, "units and tokens must be positive");
  REQUIRE(tokens < (1ll << 31) - 65536, SIKV_EUNSUPPORTED, "tokens must fit in int32");
  REQUIRE(tokens <= (1ll << 25), SIKV_EUNSUPPORTED, "fast decode supports at most 2^25 tokens per unit");
  REQUIRE(gq >= 1 && gq <= 8, SIKV_EUNSUPPORTED, "fast decode supports 1..8 query heads per KV head");
  REQUIRE(k >= 0, SIKV_EINVAL, "k must be non-negative");
  REQUIRE(sinks >= 0 && sinks <= tokens, SIKV_EINVAL, "sink count out of range");
  REQUIRE(sinks == 0 || sink_idx, SIKV_EINVAL, "sinks need sink_idx");
  REQUIRE(recent >= 0, SIKV_EINVAL, "recent count out of range");
  REQUIRE(sinks + recent == 0 || forced_frag, SIKV_EINVAL, "forced rows need forced_frag");
  REQUIRE(sinks + recent <= 16 * frag_blocks, SIKV_EINVAL, "forced rows exceed frag_blocks");
  const int64_t keff = std::min<int64_t>(k, tokens - sinks);
  REQUIRE(sinks + keff + (recent_n ? 0 : recent) >= 1, SIKV_EINVAL, "selection is empty");
  REQUIRE(!sel || sel_stride >= sinks + keff + recent, SIKV_EINVAL, "sel_stride too small");
  // kernel: 0 = auto, 1 = one CTA per unit, 3 = split units (a CTA cluster per unit),
  // 4 = two kernels (selection with two unit groups per SM, then attention)
  REQUIRE(kernel == 0 || kernel == 1 || kernel == 3 || kernel == 4, SIKV_EINVAL, "kernel must be 0, 1, 3 or 4");
  REQUIRE(lut_mode >= 0 && lut_mode <= 3, SIKV_EINVAL, "mode bits: 1 = sign-only LUT, 2 = 16-bit records");
  const bool rec16 = (lut_mode & 2) != 0;
  REQUIRE(!rec16 || kernel == 0 || kernel == 4, SIKV_EUNSUPPORTED, "16-bit records run on the two-kernel path (kernel 0 or 4)");
  // auto (measured, tools/dispatch_sweep.py): the one-CTA kernel while its units fill at most
  // one wave (two when two CTAs fit an SM: wave quantisation then still beats the two-kernel
  // path's per-unit cost), the split kernel for few long units, the two-kernel path otherwise
  bool auto_two = false, auto_split = false;
  if (kernel == 0) {
    const int c1 = decode_layout(tokens, k, sinks, gq, sikv_decode_default_cap(tokens, k, sinks)).total <= 113 * 1024
                       ? 2 : 1;
    const double waves1 = (double)units / ((double)num_sms() * c1);
    auto_split = units <= num_sms() / 2 && tokens >= 16384;
    auto_two = rec16 || (!auto_split && !(waves1 <= 1.0 || (c1 >= 2 && waves1 <= 2.0)));
  }
  if (kernel == 4 || auto_two) {
    const int64_t ke = std::min<int64_t>(k, std::max<int64_t>(tokens - sinks, 0));
    const int floor_cap = (int)std::max<int64_t>(ke + ke * 2 / 5 + 512, 1024);
    int tcap = cap > 0 ? cap : (int)std::max<int64_t>(2 * ke + 1024, 1024);
    // the selection kernel streams 64 KB of sign records per SM in flight through L1: keep
    // its shared memory at or below the 164 KB carveout (L1 >= 92 KB) while the candidate
    // buffer stays >= 1.5 k + 1024 (no segment overflow at the sampled threshold)
    const int soft_cap = (int)std::max<int64_t>(ke + ke / 2 + 1024, floor_cap);
    while (cap <= 0 && tcap > soft_cap && two_select_smem_bytes(tokens, k, sinks, tcap, gq) > 164 * 1024) tcap -= 64;
    while (cap <= 0 && tcap > floor_cap && two_select_smem_bytes(tokens, k, sinks, tcap, gq) > max_smem()) tcap -= 64;
    const bool fits = two_select_smem_bytes(tokens, k, sinks, tcap, gq) <= max_smem() &&
                      two_attend_smem_bytes(tokens, k, sinks, gq, rec16) <= max_smem();
    const bool ws_ok = workspace && workspace_bytes >= two_workspace_bytes(units, tokens, k, sinks);
    if (fits && ws_ok) {
      g_last_decode_kernel = 4;
      return cuda_ret(launch_decode_two(signs_fast, recs_fast, cent32, alpha32, sink_idx, sinks, forced_frag,
                                        frag_blocks, recent_n, recent, q, units, tokens, gq, k, tcap, out, lse, sel,
                                        sel_stride, sel_count, diag, workspace, num_sms(), unit_map, lut_mode,
                                        xchg, (cudaStream_t)stream),
                      "sikv_decode_step");
    }
    REQUIRE(kernel != 4 && !rec16, SIKV_EUNSUPPORTED,
            fits ? "the two-kernel path needs sikv_decode_workspace_bytes_k of workspace"
                 : "the two-kernel path does not fit this configuration");
  }
  // few long units: split each across a cluster of 2 / 4 / 8 CTAs so every SM has work
  if (kernel == 3 || auto_split) {
    int pick = 0, pick_cap = 0;
    for (int ns : {2, 4, 8}) {
      if ((tokens + 255) / 256 < (kernel == 3 ? 1 : 4) * ns) break;   // chunks per CTA
      const int c = cap > 0 ? cap : split_default_cap(tokens, k, sinks, ns);
      const int need = split_smem_bytes(tokens, k, sinks, gq, c, ns);
      if (need > max_smem()) continue;
      const bool two_per_sm = need <= 113 * 1024;
      if (!pick || (two_per_sm && units * ns <= 2 * num_sms()) ||
          (two_per_sm && split_smem_bytes(tokens, k, sinks, gq, pick_cap, pick) > 113 * 1024)) {
        pick = ns;
        pick_cap = c;
      }
      if (two_per_sm && units * ns >= num_sms()) break;
    }
    REQUIRE(pick || kernel != 3, SIKV_EUNSUPPORTED, "the split kernel does not fit this configuration");
    if (pick) {
      g_last_decode_kernel = 3;
      return cuda_ret(push(launch_decode_split(signs_fast, recs_fast, cent32, alpha32, sink_idx, sinks, forced_frag,
                                               frag_blocks, recent_n, recent, q, units, tokens, gq, k, pick_cap, pick, out,
                                               lse, sel, sel_stride, sel_count, diag, unit_map, lut_mode,
                                               (cudaStream_t)stream)),
                      "sikv_decode_step");
    }
  }
  if (cap <= 0) cap = sikv_decode_default_cap(tokens, k, sinks);
  int need = decode_layout(tokens, k, sinks, gq, cap).total;
  REQUIRE(need <= max_smem(), SIKV_EUNSUPPORTED,
          "decode shared-memory footprint " + std::to_string(need) + " B exceeds the device limit");
  int smem = 0;
  g_last_decode_kernel = 1;
  cudaError_t e = launch_decode(signs_fast, recs_fast, cent32, alpha32, sink_idx, sinks, forced_frag, frag_blocks,
                                recent_n, recent, q, units, tokens, gq, k, cap, out, lse, sel, sel_stride, sel_count, diag, unit_map,
                                lut_mode, (cudaStream_t)stream, &smem);
  return cuda_ret(push(e), "sikv_decode_step");
}

int sikv_debug_set_attend_skip(int v) {
  rt_bind();
  cudaError_t e = set_k1_skip(v);
  return cuda_ret(e, "sikv_debug_set_attend_skip");
}

int sikv_debug_set_decode_profile(void* clocks) {
  rt_bind();
  cudaError_t e = set_decode_profile((long long*)clocks);
  if (e == cudaSuccess) e = set_decode_two_profile((long long*)clocks);
  if (e == cudaSuccess) e = set_decode_split_profile((long long*)clocks);
  return cuda_ret(e, "sikv_debug_set_decode_profile");
}

int sikv_score_fast(const uint8_t* signs_fast, const float* cent32, const float* q, int gq, int64_t units,
                    int64_t tokens, int lut_mode, float* out, void* stream) {
  rt_bind();
  REQUIRE(signs_fast && cent32 && q && out, SIKV_EINVAL, "null pointer");
  REQUIRE(gq >= 1 && units >= 1 && tokens >= 1, SIKV_EINVAL, "bad shape");
  return cuda_ret(launch_score_fast(signs_fast, cent32, q, gq, units, tokens, lut_mode, out, (cudaStream_t)stream),
                  "sikv_score_fast");
}

int sikv_build_lut_f64(const double* q, const double* cent64, int64_t units, int groups, int sign_only,
                       double* out, void* stream) {
  rt_bind();
  REQUIRE(q && out && (sign_only || cent64), SIKV_EINVAL, "null pointer");
  REQUIRE(groups >= 1 && units >= 1, SIKV_EINVAL, "bad shape");
  return cuda_ret(launch_lut_f64(q, cent64, units, groups, sign_only, out, (cudaStream_t)stream),
                  "sikv_build_lut_f64");
}

int sikv_score_f64(const double* lut, const uint8_t* codes_ref, int64_t units, int groups, int64_t tokens,
                   double* out, void* stream) {
  rt_bind();
  REQUIRE(lut && codes_ref && out, SIKV_EINVAL, "null pointer");
  REQUIRE(groups >= 1 && groups <= 128, SIKV_EUNSUPPORTED, "groups must be 1..128");
  return cuda_ret(launch_score_f64(lut, codes_ref, units, groups, tokens, out, (cudaStream_t)stream),
                  "sikv_score_f64");
}

size_t sikv_topk_workspace_bytes(int64_t units, int64_t tokens) { return topk_workspace_bytes(units, tokens); }

static size_t a256h(size_t x) { return (x + 255) & ~(size_t)255; }

size_t sikv_window_sinks_workspace_bytes(int64_t units, int64_t tokens, int window) {
  return a256h(snap_workspace_bytes(units, tokens, window)) + a256h(topk_workspace_bytes(units, tokens)) +
         a256h((size_t)units * 2 * 4);
}

int sikv_window_sinks(const void* keys, int in_dtype, int64_t units, int64_t tokens, int64_t dim, const double* mu64,
                      const double* window, int window_n, int count, int pool_width, int32_t* sink_idx,
                      void* workspace, size_t workspace_bytes, void* stream) {
  rt_bind();
  REQUIRE(keys && mu64 && window && sink_idx && workspace, SIKV_EINVAL, "null pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "in_dtype must be 0 (f32), 1 (f64) or 2 (bf16)");
  REQUIRE(units >= 0 && tokens >= 1, SIKV_EINVAL, "keys must have at least one row");
  REQUIRE(dim >= 4 && dim % 4 == 0 && dim <= 512, SIKV_EUNSUPPORTED, "window sinks support dim % 4 == 0, <= 512");
  REQUIRE(window_n >= 1 && window_n <= 64, SIKV_EUNSUPPORTED, "window sinks support 1..64 window queries");
  REQUIRE(count >= 1 && count < tokens, SIKV_EINVAL, "count must be in [1, tokens)");
  REQUIRE(pool_width >= 1, SIKV_EINVAL, "pool_width must be positive");
  REQUIRE(tokens < (1ll << 31) - 65536, SIKV_EUNSUPPORTED, "tokens must fit in int32");
  REQUIRE(workspace_bytes >= sikv_window_sinks_workspace_bytes(units, tokens, window_n), SIKV_EINVAL,
          "workspace too small");
  if (units == 0) return SIKV_OK;
  double* pooled = nullptr;
  cudaError_t e = launch_snap_pooled(keys, in_dtype, units, tokens, (int)dim, mu64, window, window_n, pool_width,
                                     workspace, &pooled, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_ret(e, "sikv_window_sinks");
  char* p = reinterpret_cast<char*>(workspace) + a256h(snap_workspace_bytes(units, tokens, window_n));
  int32_t* counts = reinterpret_cast<int32_t*>(p + a256h(topk_workspace_bytes(units, tokens)));
  return cuda_ret(launch_topk(pooled, 0, units, tokens, nullptr, 0, count, p, sink_idx, count, counts,
                              (cudaStream_t)stream),
                  "sikv_window_sinks");
}

int sikv_topk(const void* scores, int scores_f32, int64_t units, int64_t tokens, const int32_t* forced,
              int nforced, int k, void* workspace, int32_t* out, int out_stride, int32_t* counts, void* stream) {
  rt_bind();
  REQUIRE(scores && workspace && out && counts, SIKV_EINVAL, "null pointer");
  REQUIRE(k >= 0, SIKV_EINVAL, "k must be non-negative");
  REQUIRE(nforced >= 0 && (nforced == 0 || forced), SIKV_EINVAL, "bad forced list");
  REQUIRE(tokens >= 0 && tokens < (1ll << 31) - 65536, SIKV_EUNSUPPORTED, "tokens must fit in int32");
  const int64_t need = std::min<int64_t>(k, tokens - nforced) + nforced;
  REQUIRE(out_stride >= need, SIKV_EINVAL, "out_stride too small");
  if (tokens == 0) return SIKV_OK;
  return cuda_ret(launch_topk(scores, scores_f32, units, tokens, forced, nforced, k, workspace, out, out_stride,
                              counts, (cudaStream_t)stream),
                  "sikv_topk");
}

static RefPlanes make_planes(const uint8_t* codes_ref, const uint8_t* kq_ref, const uint16_t* kq_scales,
                             const uint16_t* kq_zeros, const uint8_t* vq_ref, const uint16_t* vq_scales,
                             const uint16_t* vq_zeros, const double* kfull, const double* vfull,
                             const double* alpha64, int bits, int gs, int siq, int64_t L, int64_t D) {
  RefPlanes p{codes_ref, kq_ref, (const __half*)kq_scales, (const __half*)kq_zeros, vq_ref,
              (const __half*)vq_scales, (const __half*)vq_zeros, kfull, vfull, alpha64, bits, gs, siq,
              (int)D, L, 0, 0, 0, 0, 0};
  auto lg2 = [](int v) { int r = 0; while (v > 1) { v >>= 1; ++r; } return r; };
  if (bits >= 1 && bits <= 8 && gs > 0) {
    p.lbits = lg2(bits);
    p.lper = 3 - p.lbits;               // 8 / bits elements per byte
    p.lgs = lg2(gs);
    p.payb = (int)((D * bits + 7) / 8);
    p.ngroups = (int)(D / gs);
  }
  return p;
}

static int check_planes(const RefPlanes& p) {
  if (p.bits == 16) {
    REQUIRE(p.kfull && p.vfull, SIKV_EINVAL, "lossless planes missing");
  } else {
    REQUIRE(good_bits(p.bits) && good_group(p.gs) && p.D % p.gs == 0, SIKV_EINVAL, "bad bits/group_size");
    REQUIRE(p.kq && p.ks && p.kz && p.vq && p.vs && p.vz, SIKV_EINVAL, "quantized planes missing");
    REQUIRE(!p.siq || (p.codes && p.alpha), SIKV_EINVAL, "sign codes / alpha missing");
  }
  return SIKV_OK;
}

int sikv_dequant_rows(const uint8_t* codes_ref, const uint8_t* kq_ref, const uint16_t* kq_scales,
                      const uint16_t* kq_zeros, const uint8_t* vq_ref, const uint16_t* vq_scales,
                      const uint16_t* vq_zeros, const double* kfull, const double* vfull, const double* alpha64,
                      int bits, int group_size, int sign_in_quant, int64_t units, int64_t tokens, int64_t dim,
                      const int64_t* rows, int64_t n, int which, double* out, void* stream) {
  rt_bind();
  RefPlanes p = make_planes(codes_ref, kq_ref, kq_scales, kq_zeros, vq_ref, vq_scales, vq_zeros, kfull, vfull,
                            alpha64, bits, group_size, sign_in_quant, tokens, dim);
  if (which == 0 && bits != 16) {
    REQUIRE(vq_ref && vq_scales && vq_zeros, SIKV_EINVAL, "value planes missing");
  } else {
    int rc = check_planes(p);
    if (rc) return rc;
  }
  REQUIRE(n >= 0 && (n == 0 || (rows && out)), SIKV_EINVAL, "bad rows");
  return cuda_ret(launch_dequant_rows(p, units, rows, n, which, out, (cudaStream_t)stream), "sikv_dequant_rows");
}

size_t sikv_attend_f64_workspace_bytes(int64_t units, int heads, int sel_stride) {
  const int64_t uh = units * heads;
  return (size_t)(uh * sel_stride + uh * ATT_SPLIT * 130) * sizeof(double) + (size_t)uh * sizeof(uint32_t);
}

int sikv_attend_f64(const uint8_t* codes_ref, const uint8_t* kq_ref, const uint16_t* kq_scales,
                    const uint16_t* kq_zeros, const uint8_t* vq_ref, const uint16_t* vq_scales,
                    const uint16_t* vq_zeros, const double* kfull, const double* vfull, const double* alpha64,
                    int bits, int group_size, int sign_in_quant, int64_t units, int64_t tokens, int64_t dim,
                    const double* q, int heads, const int32_t* sel, const int32_t* nsel, int sel_stride,
                    const int32_t* sink_idx, int sinks, const double* sink_k, const double* sink_v,
                    const double* recent_k, const double* recent_v, int64_t rcap, double* ws, double* out,
                    double* chk, void* stream) {
  rt_bind();
  RefPlanes p = make_planes(codes_ref, kq_ref, kq_scales, kq_zeros, vq_ref, vq_scales, vq_zeros, kfull, vfull,
                            alpha64, bits, group_size, sign_in_quant, tokens, dim);
  int rc = check_planes(p);
  if (rc) return rc;
  REQUIRE(q && sel && nsel && ws && out && heads >= 1, SIKV_EINVAL, "null pointer");
  REQUIRE(sinks == 0 || (sink_idx && sink_k && sink_v), SIKV_EINVAL, "sink rows missing");
  REQUIRE(dim <= 128, SIKV_EUNSUPPORTED, "sparse attention supports dim <= 128");
  // ws: [U][H][sel_stride] weights | [U][H][ATT_SPLIT][130] partials | [U][H] counters
  const int64_t uh = units * heads;
  double* part = ws + uh * sel_stride;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(part + uh * ATT_SPLIT * 130);
  AttendArgs a{p, q, heads, sel, nsel, sel_stride, sink_idx, sinks, sink_k, sink_v, recent_k, recent_v,
               rcap, ws, part, cnt, out, chk};
  return cuda_ret(launch_attend_f64(a, units, (cudaStream_t)stream), "sikv_attend_f64");
}

int sikv_center(const void* x, int in_dtype, int64_t units, int64_t tokens, int64_t dim, const double* mu64,
                double* out, void* stream) {
  rt_bind();
  REQUIRE(x && mu64 && out, SIKV_EINVAL, "null pointer");
  REQUIRE(good_dtype(in_dtype), SIKV_EINVAL, "bad in_dtype");
  return cuda_ret(launch_center(x, in_dtype, units, tokens, (int)dim, mu64, out, (cudaStream_t)stream),
                  "sikv_center");
}

}  // extern "C"
