"""Pin the tcgen05 descriptor encodings in isolation (diag single-tile GEMM)
against torch.matmul in fp32 on the same bf16 inputs."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [64, 128])
@pytest.mark.parametrize("k", [64, 128])
@pytest.mark.parametrize("a_tmem", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
def test_umma_tile(n, k, a_tmem, b_mn):
    from paper_2511_08083_b200.api import diag_umma
    g = torch.Generator(device="cuda").manual_seed(1000 * n + k + 7 * a_tmem + 3 * b_mn)
    a = torch.randn(128, k, device="cuda", generator=g).to(torch.bfloat16)
    if b_mn:
        b = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
        ref = a.float() @ b.float()
    else:
        b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
        ref = a.float() @ b.float().T
    d = diag_umma(a, b, n, k, a_tmem, b_mn)
    torch.cuda.synchronize()
    err = (d - ref).abs().max().item()
    assert err < 1e-3, f"max err {err}"
