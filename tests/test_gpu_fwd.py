"""Forward parity: CUDA path (through the C ABI) vs the fp64 oracle,
element by element, O max-abs <= 2e-2 and LSE max-abs <= 2e-2."""
import numpy as np
import pytest
import torch

import oracle
from util import TOL_MAXABS, gen, np64

pytestmark = pytest.mark.gpu

CASES = [
    # B, N, Hq, Hkv, d
    (1, 128, 2, 2, 64),     # C1 (one tile: the second Q tile of the pair is empty)
    (2, 384, 4, 2, 128),    # 3 tiles: ragged pair tail, GQA G=2
    (1, 640, 8, 1, 64),     # 5 tiles, G=8
    (1, 512, 2, 2, 128),
    (2, 256, 6, 3, 64),
    (1, 200, 4, 2, 128),    # ragged: N % 128 != 0 (last tile 72 rows)
    (2, 333, 2, 1, 64),     # ragged, 3 tiles, G=2
    (1, 77, 2, 2, 128),     # a single partial tile
    (1, 1, 2, 1, 64),       # N = 1
]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("B,N,Hq,Hkv,d", CASES)
def test_fwd_parity(B, N, Hq, Hkv, d, causal):
    from paper_2511_08083_b200 import attn_fwd
    x = gen(B, N, Hq, Hkv, d, seed=N + d)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    torch.cuda.synchronize()
    O, L = oracle.attn_fwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), causal)
    eo = np.abs(np64(o) - O).max()
    el = np.abs(np64(lse) - L).max()
    assert eo <= TOL_MAXABS and el <= TOL_MAXABS, f"O err {eo}, LSE err {el}"


@pytest.mark.parametrize("causal", [False, True])
def test_fwd_stress_std4(causal):
    """Q, K ~ N(0, 4^2), V ~ N(0, 1): large running-max jumps exercise the O
    rescale path. Not a BASELINE config: the softmax is nearly one-hot, so O
    reproduces single V entries up to |O| ~ 4.5 whose bf16 output rounding alone
    is up to 2^-9 |O| (0.0156 at |O| in [4, 8)); the bound is 2e-2 plus one bf16
    ulp of the reference value, elementwise."""
    from paper_2511_08083_b200 import attn_fwd
    x = gen(1, 512, 2, 1, 128, seed=3, std_qk=4.0)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    torch.cuda.synchronize()
    O, L = oracle.attn_fwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), causal)
    excess = np.abs(np64(o) - O) - (TOL_MAXABS + np.abs(O) * 2.0 ** -8)
    el = np.abs(np64(lse) - L).max()
    assert excess.max() <= 0 and el <= TOL_MAXABS, f"O excess {excess.max()}, LSE err {el}"
