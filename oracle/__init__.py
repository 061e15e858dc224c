"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY; see ragged_oracle.py header)."""
from .ragged_oracle import (  # noqa: F401
    as_f64, scan, pack, attention_one, softmax_weights, attention, unpack,
    pack_attend_unpack, attention_image_head, l2_scores, keep_topk_l2, evit_logits, keep_evit, e4m3_decode, attention_fp8,
)
from .vit_block import (  # noqa: F401
    LN_EPS, layer_norm, gelu, linear, vit_block, vit_block_stages,
)
