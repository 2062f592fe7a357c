"""Attention tolerances of the fused path, set from the measured maxima
(profiles/round2/attention_error.json, tools/att_error.py on a B200: fp16 mma operands, fp32
accumulation, vs the float64 oracle on the same selection; every fast-path variant):

  context <= 4K    max rel-L2 measured 0.89e-3 (2-bit sign-in-quant)        -> bar 1.5e-3
  context <= 32K   max rel-L2 measured 1.39e-3 (2-bit), 2.25e-3 (1-bit),
                   2.70e-3 (direct keys, one head in the variant tests)     -> bar 3e-3
  context  > 32K   max rel-L2 measured 1.93e-3 (128K, k 4096)               -> bar 3e-3
  cosine           min measured 0.9999981                                    -> bar 0.999995
"""

ATT_COS = 0.999995


def att_rel_l2(tokens: int) -> float:
    return 1.5e-3 if tokens <= 4096 else 3e-3
