"""fp64 CPU oracles for fused attention forward/backward, the BF16 GEMM and the
memory-bound dropout-residual-LayerNorm and rotary kernels and the ring-attention LSE
merge (HipKittens, arXiv 2511.08083).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_2511_08083_b200`) never imports it and shares no code
with it: no kernels, headers, helpers, constants or pre/post-processing.

Pinned by `tests/test_oracle_*.py` (closed forms, invariants, finite
differences, a library special case and the paper's printed constants).
No function here is "parity unpinned".
"""
from .attention import (  # noqa: F401
    LN2,
    LOG2E,
    attn_fwd,
    attn_fwd_bwd,
    attn_naive,
    attn_varlen_fwd_bwd,
    attn_rows,
    attn_key_rows,
    softmax_scale,
)
from .gemm import gemm_abt, gemm_abt_rows, gemm_loops  # noqa: F401,E402
from .membound import dropout_keep, layernorm_dropout_residual, rope, rope_tables  # noqa: F401,E402
from .ring import attn_merge  # noqa: F401,E402
