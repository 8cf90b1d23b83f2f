"""Pins for oracle/membound.py: library special cases, closed forms and
invariants that do not re-type the oracle's formulas."""
import numpy as np
import torch

from oracle import dropout_keep, layernorm_dropout_residual, rope, rope_tables


def test_layernorm_matches_torch_fp64_without_dropout():
    rng = np.random.default_rng(0)
    x, res = rng.standard_normal((7, 256)), rng.standard_normal((7, 256))
    w, b = rng.standard_normal(256), rng.standard_normal(256)
    o, r = layernorm_dropout_residual(x, res, w, b, p=0.0, round_resid=False)
    ref = torch.nn.functional.layer_norm(torch.tensor(x + res), (256,), torch.tensor(w), torch.tensor(b), eps=1e-5)
    np.testing.assert_allclose(o, ref.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(r, x + res)


def test_layernorm_constant_row_gives_bias():
    """A constant row has zero deviation: o = b exactly."""
    x = np.zeros((2, 128))
    res = np.full((2, 128), 3.0)
    b = np.linspace(-1, 1, 128)
    o, _ = layernorm_dropout_residual(x, res, np.ones(128), b, p=0.0)
    np.testing.assert_array_equal(o, np.tile(b, (2, 1)))


def test_layernorm_normalised_moments():
    """With w = 1, b = 0 each output row has mean 0 and variance var/(var+eps)."""
    rng = np.random.default_rng(1)
    x, res = rng.standard_normal((5, 512)) * 3, rng.standard_normal((5, 512))
    o, r = layernorm_dropout_residual(x, res, np.ones(512), np.zeros(512), p=0.0)
    var = r.var(axis=1)
    np.testing.assert_allclose(o.mean(axis=1), 0, atol=1e-12)
    np.testing.assert_allclose(o.var(axis=1), var / (var + 1e-5), rtol=1e-10)


def test_dropout_keep_rate_and_determinism():
    k = dropout_keep(1 << 20, 0.25, seed=5)
    assert abs(k.mean() - 0.75) < 3e-3  # binomial sd ~4e-4
    np.testing.assert_array_equal(k, dropout_keep(1 << 20, 0.25, seed=5))
    assert (k != dropout_keep(1 << 20, 0.25, seed=6)).mean() > 0.3
    np.testing.assert_array_equal(dropout_keep(100, 0.25, seed=5, offset=1000), k[1000:1100])
    assert dropout_keep(10, 0.0, seed=1).all()


def test_dropout_hash_brute_force():
    """The vectorised hash equals the plain-integer lowbias32 hash, element by element."""
    M = (1 << 32) - 1

    def keep1(i, p, seed):
        x = (i * 0x9E3779B9 + seed) & M
        x ^= x >> 16
        x = (x * 0x7FEB352D) & M
        x ^= x >> 15
        x = (x * 0x846CA68B) & M
        x ^= x >> 16
        return x >= int(p * 2 ** 32)

    k = dropout_keep(300, 0.4, seed=123)
    assert all(k[i] == keep1(i, 0.4, 123) for i in range(300))


def test_layernorm_dropout_residual_output():
    rng = np.random.default_rng(2)
    x, res = rng.standard_normal((3, 128)), rng.standard_normal((3, 128))
    _, r = layernorm_dropout_residual(x, res, np.ones(128), np.zeros(128), p=0.5, seed=9, round_resid=False)
    keep = dropout_keep(3 * 128, 0.5, 9).reshape(3, 128)
    np.testing.assert_allclose(r, res + np.where(keep, 2 * x, 0), rtol=0, atol=0)


def test_rope_identity_at_position_zero_and_norm_preserving():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 5, 3, 64))
    c, s = rope_tables(5, 64)
    y = rope(x, c, s)
    np.testing.assert_allclose(y[:, 0], x[:, 0], rtol=0, atol=0)  # theta = 0
    pair = lambda a: a[..., :32] ** 2 + a[..., 32:] ** 2
    np.testing.assert_allclose(pair(y), pair(x), rtol=1e-12)


def test_rope_equals_complex_rotation_and_inverts():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1, 7, 2, 16))
    c, s = rope_tables(7, 16)
    z = (x[..., :8] + 1j * x[..., 8:]) * np.exp(1j * np.arctan2(s, c))[None, :, None, :]
    y = rope(x, c, s)
    np.testing.assert_allclose(y[..., :8], z.real, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y[..., 8:], z.imag, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(rope(y, c, -s), x, rtol=1e-12, atol=1e-12)


def test_rope_attention_gradient_chain_rule_finite_differences():
    """Reading #21 + NEXT #3 (attention on rotated Q, K): the gradient w.r.t. the unrotated Q, K is
    the inverse rotation of the oracle's gradient w.r.t. the rotated ones, R^T g = rope(g, c, -s)
    (what attn_bwd_rope computes). Pinned by central finite differences of L = sum(O * dO)."""
    from oracle import attn_fwd, attn_fwd_bwd
    rng = np.random.default_rng(11)
    B, N, Hq, Hkv, d = 1, 5, 2, 1, 8
    Q, K, V, dO = (rng.standard_normal(s) for s in ((B, N, Hq, d), (B, N, Hkv, d), (B, N, Hkv, d), (B, N, Hq, d)))
    c, s = rope_tables(N, d)
    for causal in (False, True):
        ref = attn_fwd_bwd(rope(Q, c, s), rope(K, c, s), V, dO, causal)
        gq, gk = rope(ref["dQ"], c, -s), rope(ref["dK"], c, -s)
        loss = lambda q, k: float((attn_fwd(rope(q, c, s), rope(k, c, s), V, causal)[0] * dO).sum())
        h = 1e-6
        for (t, g) in ((Q, gq), (K, gk)):
            for idx in [(0, 0, 0, 0), (0, 3, 0, 5), (0, 4, t.shape[2] - 1, 7), (0, 2, 0, 2)]:
                tp, tm = t.copy(), t.copy()
                tp[idx] += h
                tm[idx] -= h
                fd = (loss(tp, K) - loss(tm, K)) / (2 * h) if t is Q else (loss(Q, tp) - loss(Q, tm)) / (2 * h)
                assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(fd)), (causal, idx, fd, g[idx])
