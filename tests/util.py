"""Shared helpers for GPU parity tests: run the CUDA path, compare with the
fp64 oracle on the same (D2H-copied) bf16 inputs at the BASELINE tolerances:
max-abs 2e-2 on O and LSE, relative L2 1e-2 on dQ, dK, dV."""
import numpy as np

from paper_2511_08083_b200.inputs import make_inputs

TOL_MAXABS = 2e-2
TOL_RELL2 = 1e-2


def np64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def rel_l2(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


def gen(B, N, Hq, Hkv, d, seed=0, std_qk=None):
    return make_inputs(B, N, Hq, Hkv, d, seed=seed, device="cuda", std_qk=std_qk)
