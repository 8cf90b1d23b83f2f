"""Python binding validation (CPU: every check fires before any CUDA call)."""
import pytest
import torch

from paper_2511_08083_b200 import api


def t(*shape, dtype=torch.bfloat16):
    return torch.zeros(*shape, dtype=dtype)


def test_rejects_cpu_and_bad_dtype_and_layout():
    q, k, v = t(1, 128, 2, 64), t(1, 128, 2, 64), t(1, 128, 2, 64)
    with pytest.raises(ValueError, match="CUDA"):
        api.attn_fwd(q, k, v)
    with pytest.raises(ValueError):
        api._check_tensor("q", t(2, 2, dtype=torch.float32))
    with pytest.raises(ValueError):
        api._shapes(t(1, 128, 2, 64), t(1, 64, 2, 64), t(1, 32, 2, 64))  # k, v differ
    with pytest.raises(ValueError):
        api._shapes(t(1, 128, 2, 64), t(1, 128, 2, 32), t(1, 128, 2, 32))
    with pytest.raises(ValueError):
        api._shapes(t(1, 128, 2, 64), t(2, 128, 2, 64), t(2, 128, 2, 64))
    assert api._shapes(t(2, 256, 8, 128), t(2, 256, 2, 128), t(2, 256, 2, 128)) == (2, 256, 256, 8, 2, 128)
    assert api._shapes(t(2, 100, 8, 64), t(2, 300, 2, 64), t(2, 300, 2, 64)) == (2, 100, 300, 8, 2, 64)


def test_varlen_binding_validation():
    q, k = t(10, 4, 64), t(12, 2, 64)
    cu = torch.tensor([0, 4, 10], dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        api.attn_fwd_varlen(q, k, k, cu, cu, 6, 8)
    with pytest.raises(ValueError):
        api._check_tensor("cu", cu.to(torch.int64), torch.int32)


def test_library_missing_is_loud(monkeypatch, tmp_path):
    from paper_2511_08083_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "_LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="not built"):
        _lib.lib()


def test_check_cu_seqlens():
    cu = lambda *v: torch.tensor(v, dtype=torch.int32)
    api.check_cu_seqlens(cu(0, 3, 3, 10), cu(0, 5, 9, 9), 10, 9, 7, 5)
    with pytest.raises(ValueError, match="rise"):
        api.check_cu_seqlens(cu(0, 3, 2, 10), cu(0, 5, 9, 9), 10, 9, 8, 5)
    with pytest.raises(ValueError, match="rise"):
        api.check_cu_seqlens(cu(0, 3, 3, 10), cu(0, 5, 9, 9), 11, 9, 8, 5)
    with pytest.raises(ValueError, match="max_seqlen_q"):
        api.check_cu_seqlens(cu(0, 3, 3, 10), cu(0, 5, 9, 9), 10, 9, 6, 5)


def test_caller_buffer_shapes_are_checked():
    """Caller-supplied outputs / workspaces reach the C ABI as raw pointers: a wrongly
    shaped one must be a ValueError in the binding, not an out-of-bounds write."""
    api._expect_shape("out", t(1, 128, 2, 64), (1, 128, 2, 64))
    with pytest.raises(ValueError, match="shape"):
        api._expect_shape("out", t(1, 128, 2, 32), (1, 128, 2, 64))
    with pytest.raises(ValueError, match="shape"):
        api._expect_shape("lse", t(1, 2, 127, dtype=torch.float32), (1, 2, 128))
