"""B200-native (sm_100a) self-indexing KV cache (arXiv 2603.14224).

Drop-in for the reference package's API (``sikv``): the same names are exported here and
run on the GPU through ``libsikv_b200.so``.  The batched decode hot path is in
:mod:`paper_2603_14224_b200.batch`.
"""

from .api import (  # noqa: F401
    AttentionOutput,
    CacheConfig,
    Codebook,
    ErrorReport,
    LookupTable,
    MemoryReport,
    NormalizationState,
    OpCounters,
    QuantConfig,
    QuantizedTensor,
    SelfIndexingCache,
    SignCodeMatrix,
    TokenSelection,
    append_token,
    apply_normalization,
    build_codebook,
    build_lut,
    build_sign_lut,
    collect,
    compute_channel_stats,
    dense_scores,
    dequantize_keys,
    dequantize_values,
    encode_keys,
    encode_sign_code,
    exact_attention,
    memory_report,
    memory_report_from_shapes,
    output_error,
    prefill,
    quantize_key_magnitudes,
    quantize_values,
    resolve_dynamic_k,
    score_tokens,
    select_sink_tokens,
    select_tokens,
    sign_entropy,
    sign_pattern_vectors,
    sparse_attention,
    top_k_select,
)

__version__ = "0.1.0"

__all__ = [
    "AttentionOutput", "CacheConfig", "Codebook", "ErrorReport", "LookupTable", "MemoryReport",
    "NormalizationState", "OpCounters", "QuantConfig", "QuantizedTensor", "SelfIndexingCache",
    "SignCodeMatrix", "TokenSelection", "append_token", "apply_normalization", "build_codebook",
    "build_lut", "build_sign_lut", "collect", "compute_channel_stats", "dense_scores",
    "dequantize_keys", "dequantize_values", "encode_keys", "encode_sign_code", "exact_attention",
    "memory_report", "memory_report_from_shapes", "output_error", "prefill", "quantize_key_magnitudes",
    "quantize_values", "resolve_dynamic_k", "score_tokens", "select_sink_tokens", "select_tokens",
    "sign_entropy", "sign_pattern_vectors", "sparse_attention", "top_k_select",
]
