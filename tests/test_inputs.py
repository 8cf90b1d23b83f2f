"""Seeded input generator: determinism and per-batch independence (the
property the multi-GPU batch split relies on)."""
import torch

from paper_2511_08083_b200.inputs import make_inputs, sample_rows, splitmix64


def test_deterministic_and_bf16():
    a = make_inputs(2, 16, 4, 2, 8, seed=5)
    b = make_inputs(2, 16, 4, 2, 8, seed=5)
    for k in a:
        assert a[k].dtype == torch.bfloat16
        assert torch.equal(a[k], b[k])
    c = make_inputs(2, 16, 4, 2, 8, seed=6)
    assert not torch.equal(a["Q"], c["Q"])


def test_batch_subset_matches_full():
    full = make_inputs(4, 8, 4, 2, 8, seed=1)
    part = make_inputs(4, 8, 4, 2, 8, seed=1, batches=[2, 3])
    for k in full:
        assert torch.equal(full[k][2:4], part[k])


def test_distribution_roughly_standard_normal():
    x = make_inputs(1, 512, 4, 1, 64, seed=0)["Q"].float()
    assert abs(x.mean().item()) < 0.02 and abs(x.std().item() - 1.0) < 0.02


def test_splitmix_and_rows():
    assert splitmix64(0, 1) != splitmix64(1, 0)
    rows = sample_rows(1024, 64, seed=0)
    assert rows == sorted(set(rows)) and 0 in rows and 1023 in rows and len(rows) == 64
