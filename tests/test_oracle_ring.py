"""Pins for the ring-attention LSE merge oracle (oracle/ring.py): merging the
attention results over two disjoint key sets must equal the attention over
their union computed in one piece by the (already pinned) attention oracle —
an identity of the softmax, not a restatement of the merge formula — plus the
empty-partial identity, symmetry and the all-empty row."""
import numpy as np
import pytest

from oracle import attn_fwd, attn_merge


def rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


@pytest.mark.parametrize("split", [1, 7, 20, 39])
def test_merge_of_disjoint_key_sets_equals_union(split):
    B, Nq, Nk, Hq, Hkv, d = 2, 9, 40, 4, 2, 8
    Q, K, V = rand((B, Nq, Hq, d), 1), rand((B, Nk, Hkv, d), 2), rand((B, Nk, Hkv, d), 3)
    O, L = attn_fwd(Q, K, V, False)
    O1, L1 = attn_fwd(Q, K[:, :split], V[:, :split], False)
    O2, L2 = attn_fwd(Q, K[:, split:], V[:, split:], False)
    Om, Lm = attn_merge(O1, L1, O2, L2)
    np.testing.assert_allclose(Om, O, atol=1e-13)
    np.testing.assert_allclose(Lm, L, atol=1e-13)


def test_merge_three_way_any_order():
    B, N, H, d = 1, 5, 2, 4
    Q, K, V = rand((B, N, H, d), 4), rand((B, 30, H, d), 5), rand((B, 30, H, d), 6)
    parts = [attn_fwd(Q, K[:, a:b], V[:, a:b], False) for a, b in ((0, 10), (10, 11), (11, 30))]
    O, L = attn_fwd(Q, K, V, False)
    for order in ((0, 1, 2), (2, 0, 1), (1, 2, 0)):
        Oa, La = parts[order[0]]
        for i in order[1:]:
            Oa, La = attn_merge(Oa, La, *parts[i])
        np.testing.assert_allclose(Oa, O, atol=1e-13)
        np.testing.assert_allclose(La, L, atol=1e-13)


def test_merge_with_empty_partial_and_dead_rows():
    B, N, H, d = 1, 6, 2, 4
    O1, L1 = rand((B, N, H, d), 7), rand((B, H, N), 8)
    Oe, Le = np.zeros((B, N, H, d)), np.full((B, H, N), -np.inf)
    O, L = attn_merge(O1, L1, Oe, Le)
    np.testing.assert_array_equal(O, O1)
    np.testing.assert_array_equal(L, L1)
    O, L = attn_merge(Oe, Le, O1, L1)
    np.testing.assert_array_equal(O, O1)
    O, L = attn_merge(Oe, Le, Oe, Le)
    assert np.all(O == 0) and np.all(np.isneginf(L))


def test_merge_causal_split_equals_causal():
    """Causal attention of a query block = merge of the strictly-earlier keys
    (non-causal) and its own block (causal): the ring's diagonal decomposition."""
    B, c, H, d = 1, 8, 2, 4
    Q, K, V = rand((B, 2 * c, H, d), 9), rand((B, 2 * c, H, d), 10), rand((B, 2 * c, H, d), 11)
    O, L = attn_fwd(Q, K, V, True)
    Oa, La = attn_fwd(Q[:, c:], K[:, :c], V[:, :c], False)
    Ob, Lb = attn_fwd(Q[:, c:], K[:, c:], V[:, c:], True)
    Om, Lm = attn_merge(Oa, La, Ob, Lb)
    np.testing.assert_allclose(Om, O[:, c:], atol=1e-13)
    np.testing.assert_allclose(Lm, L[:, :, c:], atol=1e-13)
