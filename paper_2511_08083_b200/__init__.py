"""B200-native (sm_100a) fused bf16 attention forward/backward.

The data-parallel hot path of HipKittens (arXiv 2511.08083): MHA/GQA,
causal and non-causal, head dim 64/128, behind the C ABI in include/hk_attn.h.
"""
from .api import (  # noqa: F401
    Attention, AttentionRope, AttentionVarlen, HKError, attn_bwd, attn_bwd_rope, attn_bwd_varlen, attn_fwd,
    attn_fwd_rope, attn_fwd_varlen, bwd_ds_workspace_bytes, bwd_workspace_bytes, default_bwd_workspace_bytes, gemm, get_max_ctas, ln_dropout_residual, rope, set_max_ctas,
    sm_budget,
)
