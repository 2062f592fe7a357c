/*
 * sikv_b200.h — C ABI of libsikv_b200.so, the B200 (sm_100a) self-indexing KV-cache path.
 *
 * The reference (arXiv 2603.14224's package, /root/reference/pkg/src/sikv) is a Python/numpy
 * package with no FFI; its boundary is the Python API in sikv/__init__.py.  These entry
 * points are what that API binds to through ctypes: every reference
 * function on the decode path maps to one call below, cited next to it.
 *
 * Conventions
 *   - all tensor arguments are DEVICE pointers, contiguous, row-major, owned by the caller
 *     (the library never allocates or frees); `stream` is a cudaStream_t (NULL = default);
 *   - calls are asynchronous on `stream`, stateless and re-entrant; argument errors are
 *     reported synchronously via the return code, device-side data errors via `status_dev`
 *     (a device int the caller zeroes and reads back: bit0 = fp16 parameter range exceeded,
 *     bit1 = alpha does not dominate |K'|, bit2 = non-finite input, bit3 = mean certificate
 *     failed and the sequential fallback ran (informational));
 *   - return 0 on success, SIKV_EINVAL / SIKV_EUNSUPPORTED / SIKV_ECUDA otherwise; the
 *     message is available from sikv_last_error() (thread-local).
 *   - in_dtype: 0 = float32, 1 = float64, 2 = bfloat16.
 *
 * Layouts ("reference layout" = the reference's packed numpy arrays, bit for bit):
 *   codes_ref  [U][L][ceil(G/2)] u8   two 4-bit sign codes per byte, low nibble = lower group
 *                                     (codebook.py:50-90, bitpack.py:27-48)
 *   kq_ref/vq_ref [U][L][ceil(D*bits/8)] u8, element e at bits (e % (8/bits))*bits of byte
 *                                     e/(8/bits) (bitpack.py:27-48)
 *   *_scales / *_zeros [U][L][D/group] fp16 (quantizer.py:52-94)
 * Fast layout (D = 128, bits = 2, group = 32, sign_in_quant): see DESIGN.md §3
 *   signs_fast [U][L][16] u8  sign plane, byte i of token t = reference byte (t+i) mod 16
 *   recs_fast  [U][L][128] u8 per-token record: K/V 2-bit payloads in mma.sync fragment
 *                             order, fp16 (scale, zero) x 4 groups for K and V, K sign words
 */
#ifndef SIKV_B200_H
#define SIKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIKV_OK 0
#define SIKV_EINVAL 1
#define SIKV_ECUDA 2
#define SIKV_EUNSUPPORTED 3

const char* sikv_last_error(void);
int sikv_abi_version(void);   /* 8 */

/* ---------------------------------------------------------------- encoder (prefill)
 * replaces: compute_channel_stats   normalize.py:56-61
 *           encode_keys             codebook.py:116-125
 *           build_codebook          codebook.py:128-160
 *           quantize_key_magnitudes quantizer.py:155-170
 *           quantize_values         quantizer.py:106-140
 *           the quantisation half of prefill, cache.py:229-245
 * what: bit0 = compute mu/alpha (else use the given mu64/alpha64), bit1 = pack + codebook.
 * bits: 1, 2, 4, 8, or 0 for lossless (codes + codebook only).  codes_in (nullable) replaces
 * the computed sign codes for the codebook (build_codebook(keys_norm, codes)). */
size_t sikv_encode_workspace_bytes(int64_t units, int64_t tokens, int64_t dim);
int sikv_encode(const void* keys, const void* values, int in_dtype, int64_t units, int64_t tokens,
                int64_t dim, int bits, int group_size, int sign_in_quant, int what,
                const uint8_t* codes_in, double* mu64, double* alpha64, float* mu32, float* alpha32,
                double* cent64, float* cent32, uint8_t* codes_ref, uint8_t* kq_ref,
                uint16_t* kq_scales, uint16_t* kq_zeros, uint8_t* vq_ref, uint16_t* vq_scales,
                uint16_t* vq_zeros, uint8_t* signs_fast, uint8_t* recs_fast, void* workspace,
                size_t workspace_bytes, int* status_dev, void* stream);

/* 16-bit fast-path records (bits = 16, "Ours (16 bits)"; cache.py:236-238 at model precision):
 * recs16 [U][L][512] u8 = K^ = (K - mu) / alpha32 and V in fp16, in the mma fragment orders of
 * DESIGN.md §3; decode with sikv_decode_step(mode bit 1).  status bit 4: V outside fp16.
 * bits 4 / 8 use the same records: the 4- / 8-bit planes from sikv_encode are dequantised by
 * sikv_dequant_rows (float64, cache.gather order) and passed here with mu64 = 0. */
int sikv_pack16(const void* keys, const void* values, int in_dtype, int64_t units, int64_t tokens,
                const double* mu64, const float* alpha32, uint8_t* recs16, int* status_dev, void* stream);

/* full-precision rows: out_k = K[idx] - mu (centred), out_v = V[idx]; float32 or float64 out.
 * replaces: sink_k / sink_v construction, cache.py:247-270 */
int sikv_gather_rows(const void* keys, const void* values, int in_dtype, int64_t units,
                     int64_t tokens, int64_t dim, const int32_t* idx, int64_t n,
                     const double* mu64, void* out_k, void* out_v, int out_f64, void* stream);

/* SnapKV-style sinks from a query window, float64 (K' = keys - mu; column softmax of
 * K' W^T / sqrt(dim) over the tokens, votes = row sums, max-pool of width pool_width with
 * edge replication, the count highest, ties -> lower index, sorted): sink_idx [U][count].
 * window [U][window_n][dim] float64; needs 1 <= count < tokens.
 * replaces: select_sink_tokens, cache.py:185-209 (prefill's query_window branch, 249-252) */
size_t sikv_window_sinks_workspace_bytes(int64_t units, int64_t tokens, int window_n);
int sikv_window_sinks(const void* keys, int in_dtype, int64_t units, int64_t tokens, int64_t dim,
                      const double* mu64, const double* window, int window_n, int count, int pool_width,
                      int32_t* sink_idx, void* workspace, size_t workspace_bytes, void* stream);

/* decode-time append of one token per unit at ring position pos (float32/64 rows only; the
 * batched fast path uses sikv_append_forced below).
 * replaces: append_token, cache.py:274-287 */
int sikv_append(const void* k, const void* v, int in_dtype, int64_t units, int64_t dim,
                const double* mu64, void* recent_k, void* recent_v, int64_t rcap, int64_t pos,
                int out_f64, int* status_dev, void* stream);

/* ---------------------------------------------------------------- fused decode step (hot path)
 * For every unit: q-bar = sum of its gq query heads, LUT + pair-table scoring of all tokens,
 * exact top-k (ties -> lower index) of the non-sink tokens, and sparse attention of each of
 * the gq heads over sinks + recents + selected tokens.
 * replaces, per unit: select_tokens(cache, sum_h q_h, k=k)   cache.py:290-309
 *                     sparse_attention(q_h, selection, cache) attention.py:52-62 (for each h)
 * out [U][gq][128] f32; lse (nullable) [U][gq]; sel (nullable) [U][sel_stride] sorted token
 * indices (sinks U recents U dynamic); sel_count (nullable) [U]; diag (nullable) [U]
 * (bits0-1 = selection mode, bit2 = exact rescoring fallback ran).
 * cap = candidate buffer entries (0 = choose); needs sikv_decode_smem_bytes <= 227 KB. */
int sikv_decode_smem_bytes(int64_t tokens, int k, int sinks, int gq, int cap);
int sikv_decode_default_cap(int64_t tokens, int k, int sinks);
size_t sikv_decode_workspace_bytes(int64_t units, int64_t tokens);
/* workspace for every decode kernel at top-k k (the two-kernel path stores the dynamic lists) */
size_t sikv_decode_workspace_bytes_k(int64_t units, int64_t tokens, int k, int sinks);
/* kernel: 0 = auto (a thread-block cluster per unit for few long units: units <= SMs / 2 and
 * tokens >= 16K; one CTA per unit while the units fill at most one wave of the SMs, or two
 * waves when two CTAs fit an SM; else the two-kernel path, given a workspace of
 * sikv_decode_workspace_bytes_k and a selection kernel that fits shared memory; its attention
 * kernel splits each unit over several CTAs when the units are fewer than four per SM),
 * 1 = one CTA per unit, 3 = split units across a cluster, 4 = force the two-kernel path
 * (selection, then attention).
 * sink_idx [U][sinks] int32: each unit's sink token indices in ascending order (as
 * select_sink_tokens / sikv_window_sinks return them); the kernels rely on the order.
 * Recent rows: recent_n (nullable) [U] int32 = recent rows of each unit (forced, scored
 * -inf: cache.py:290-309; sel then ends with tokens + 0 .. recent_n[u] - 1); recent = their
 * maximum (or the count of every unit when recent_n is NULL).
 * unit_map (nullable) [units] int32: the cache unit each query unit reads (q, out, sel, diag are
 * per query unit; the planes, sinks, recents per cache unit): the per-q-head policy runs one
 * query unit of gq = 1 per query head over its KV head's cache (cache.py:290-309 per head).
 * lut_mode (mode bits): bit 0 = sign-only LUT (build_sign_lut, retrieval.py:54-62: the code's +-1
 * pattern instead of its centroid; select_tokens(..., sign_only=True)); bit 1 = recs_fast holds
 * 16-bit records (sikv_pack16; two-kernel path only). */
int sikv_decode_step(const uint8_t* signs_fast, const uint8_t* recs_fast, const float* cent32,
                     const float* alpha32, const int32_t* sink_idx, int sinks, const uint32_t* forced_frag,
                     int frag_blocks, const int32_t* recent_n, int recent, const float* q, int64_t units,
                     int64_t tokens, int gq, int k, int cap, float* out, float* lse, int32_t* sel,
                     int sel_stride, int32_t* sel_count, int32_t* diag, void* workspace,
                     size_t workspace_bytes, const int32_t* unit_map, int lut_mode, int kernel,
                     void* stream);

/* ---------------------------------------------------------------- multi-GPU output exchange
 * The head x batch sharded decode ("NCCL over NVLink only for the final
 * output all-gather") with the all-gather fused into the decode instead: every rank's
 * attention epilogue stores its units' outputs as bf16 straight into every rank's model-layout
 * buffer over NVLink (peer pointers from CUDA IPC), then releases a per-rank arrival counter.
 * out[r] is rank r's bf16 buffer [units_total][gq][128] (row = global unit id, i.e. the
 * [layers][batch][kv_heads * gq][128] model layout); flag[r] its u64 counter; npeers <= 8
 * (this rank included); unit_gid [units] (device) the global id of each local unit.  After
 * step e (1, 2, ...) of every rank, rank r's counter reaches e * units_total * gq (rows; the
 * per-q-head policy pushes units_total * gq one-row query units): sikv_exchange_wait enqueues
 * that wait on a stream. */
#define SIKV_MAX_PEERS 8
typedef struct {
  int npeers;
  void* out[SIKV_MAX_PEERS];
  unsigned long long* flag[SIKV_MAX_PEERS];
  const int32_t* unit_gid;
} sikv_exchange;

/* sikv_decode_step plus the fused output exchange (xchg NULL or npeers 0: none).  The two-
 * kernel path stores from its attention epilogue; the other paths from one push kernel
 * launched after the decode kernel on the same stream. */
int sikv_decode_step_x(const uint8_t* signs_fast, const uint8_t* recs_fast, const float* cent32,
                       const float* alpha32, const int32_t* sink_idx, int sinks, const uint32_t* forced_frag,
                       int frag_blocks, const int32_t* recent_n, int recent, const float* q, int64_t units,
                       int64_t tokens, int gq, int k, int cap, float* out, float* lse, int32_t* sel,
                       int sel_stride, int32_t* sel_count, int32_t* diag, void* workspace,
                       size_t workspace_bytes, const int32_t* unit_map, int lut_mode, int kernel,
                       const sikv_exchange* xchg, void* stream);
/* enqueue on `stream` a wait until *flag >= target (system-scope acquire) */
int sikv_exchange_wait(const unsigned long long* flag, unsigned long long target, void* stream);
/* CUDA IPC for the peer buffers: the 64-byte handle of the allocation holding dev_ptr and
 * dev_ptr's offset in it; the mapping of another process's handle into this one (the
 * allocation's base; add the offset; peer access enabled lazily) / its release */
int sikv_ipc_handle(const void* dev_ptr, void* handle64, size_t* offset);
int sikv_ipc_open(const void* handle64, void** dev_ptr);
int sikv_ipc_close(void* dev_ptr);

/* the decode path (1, 3 or 4, as the kernel argument) the last sikv_decode_step of this host
 * thread launched; the two-kernel path (4) starts two kernels per step, the others one */
int sikv_decode_last_kernel(void);

/* forced rows (sinks then recents; float32 centred K' and V) -> the decode kernel's blocks of
 * 16 rows: forced_frag [U][frag_blocks][sikv_forced_block_words()] u32 = fp16 K^ mma
 * fragments [32][32], fp16 V fragments [32][32], 16 float32 row scales (K^ = K' /
 * (alpha-hat * scale), scale a power of two, 1 unless |K'| of a recent row exceeds the
 * prefill alpha).  Re-packs the blocks covering rows [row_begin, row_end); rows >= sinks +
 * recent_n[u] (or + recent) are zero.  status_dev (nullable): bit2 non-finite, bit4 a V entry
 * outside the fp16 range.
 * replaces: the full-precision sink / recent rows of cache.gather, cache.py:137-144 */
int sikv_forced_blocks(int sinks, int64_t rcap);
int sikv_forced_block_words(void);
int sikv_pack_forced(const float* sink_k, const float* sink_v, int sinks, const float* recent_k,
                     const float* recent_v, int64_t rcap, const int32_t* recent_n, int recent,
                     const float* alpha32, int64_t units, uint32_t* forced_frag, int frag_blocks,
                     int row_begin, int row_end, int* status_dev, void* stream);

/* decode-time append into the forced-row ring of the batched fast path: row i of k / v
 * [n][128] goes to unit unit_ids[i] (or i when unit_ids is NULL; ids distinct within a call)
 * at ring position recent_n[unit], centred in float64 with the frozen prefill mu and stored
 * as float32, the fragment block holding it is re-packed and recent_n[unit] is incremented,
 * all on the device (no host sync).  The caller guarantees recent_n[unit] < rcap (status
 * bit5 otherwise, row dropped); bit2 non-finite input, bit4 V outside the fp16 range.
 * replaces: append_token, cache.py:274-287, for every listed unit at once */
int sikv_append_forced(const void* k, const void* v, int in_dtype, int64_t n, const int32_t* unit_ids,
                       const double* mu64, const float* alpha32, const float* sink_k, const float* sink_v,
                       int sinks, float* recent_k, float* recent_v, int64_t rcap, int32_t* recent_n,
                       uint32_t* forced_frag, int frag_blocks, int* status_dev, void* stream);

/* debug: per-unit phase clocks [U][12] int64 (clock64 at phase boundaries) for every
 * subsequent sikv_decode_step; NULL disables. */
int sikv_debug_set_decode_profile(void* clocks);

/* debug: bit 0 makes the one-CTA-per-unit decode kernel skip sparse attention (phase timing
 * of the scoring / selection half alone); 0 restores normal operation. */
int sikv_debug_set_attend_skip(int bits);

/* fast-path float32 scores only (the decode kernel's scoring, for verification / API).
 * replaces: build_lut + score_tokens on the group-summed query, retrieval.py:46-77 */
int sikv_score_fast(const uint8_t* signs_fast, const float* cent32, const float* q, int gq,
                    int64_t units, int64_t tokens, int lut_mode, float* out, void* stream);

/* ---------------------------------------------------------------- reference-exact float64 API
 * replaces: build_lut retrieval.py:46-51, build_sign_lut retrieval.py:54-62 */
int sikv_build_lut_f64(const double* q, const double* cent64, int64_t units, int groups,
                       int sign_only, double* out, void* stream);
/* replaces: score_tokens retrieval.py:65-77 (numpy pairwise summation order) */
int sikv_score_f64(const double* lut, const uint8_t* codes_ref, int64_t units, int groups,
                   int64_t tokens, double* out, void* stream);
/* replaces: top_k_select retrieval.py:127-161.  forced [U][nforced] = sink U recent indices
 * (sorted, unique); out [U][out_stride] sorted; counts [U][2] = (total, dynamic). */
size_t sikv_topk_workspace_bytes(int64_t units, int64_t tokens);
int sikv_topk(const void* scores, int scores_f32, int64_t units, int64_t tokens,
              const int32_t* forced, int nforced, int k, void* workspace, int32_t* out,
              int out_stride, int32_t* counts, void* stream);
/* replaces: dequantize_values quantizer.py:143-152 (which = 0) and dequantize_keys
 * quantizer.py:173-184 / direct-key dequant (which = 1) for the given rows */
int sikv_dequant_rows(const uint8_t* codes_ref, const uint8_t* kq_ref, const uint16_t* kq_scales,
                      const uint16_t* kq_zeros, const uint8_t* vq_ref, const uint16_t* vq_scales,
                      const uint16_t* vq_zeros, const double* kfull, const double* vfull,
                      const double* alpha64, int bits, int group_size, int sign_in_quant,
                      int64_t units, int64_t tokens, int64_t dim, const int64_t* rows, int64_t n,
                      int which, double* out, void* stream);
/* replaces: sparse_attention attention.py:52-62 with cache.gather cache.py:118-158, float64.
 * ws: sikv_attend_f64_workspace_bytes(units, heads, sel_stride) bytes (the weights, then the
 * split CTAs' partials and counters); out [U][heads][dim] (dim <= 128); chk (nullable)
 * [U][heads] = the weights' sum. */
size_t sikv_attend_f64_workspace_bytes(int64_t units, int heads, int sel_stride);
int sikv_attend_f64(const uint8_t* codes_ref, const uint8_t* kq_ref, const uint16_t* kq_scales,
                    const uint16_t* kq_zeros, const uint8_t* vq_ref, const uint16_t* vq_scales,
                    const uint16_t* vq_zeros, const double* kfull, const double* vfull,
                    const double* alpha64, int bits, int group_size, int sign_in_quant,
                    int64_t units, int64_t tokens, int64_t dim, const double* q, int heads,
                    const int32_t* sel, const int32_t* nsel, int sel_stride,
                    const int32_t* sink_idx, int sinks, const double* sink_k, const double* sink_v,
                    const double* recent_k, const double* recent_v, int64_t rcap, double* ws,
                    double* out, double* chk, void* stream);
/* replaces: apply_normalization normalize.py:64-69 (out = x - mu, float64) */
int sikv_center(const void* x, int in_dtype, int64_t units, int64_t tokens, int64_t dim,
                const double* mu64, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SIKV_B200_H */
