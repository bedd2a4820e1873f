"""tcgen05 (5th-gen tensor core) row GEMM: out = A . theta (or theta^T) in
3xTF32 with the accumulator in TMEM -- checked against a float64 reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [32, 64])
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("rows", [1, 127, 128, 129, 1000, 100003])
def test_rowmm_tcgen05_matches_fp64(d, transpose, rows):
    from paper_2212_04540_b200.tensorops import mm_theta
    rng = np.random.default_rng(rows + d)
    a = rng.standard_normal((rows, d), dtype=np.float32)
    th = (rng.standard_normal((d, d)) / np.sqrt(d)).astype(np.float32)
    out = mm_theta(torch.from_numpy(a).cuda(), torch.from_numpy(th).cuda(), transpose).cpu().numpy()
    ref = a.astype(np.float64) @ (th.T if transpose else th).astype(np.float64)
    err = np.abs(out - ref).max()
    assert err <= 2e-5 * np.abs(ref).max() + 1e-6, err
    # deterministic
    out2 = mm_theta(torch.from_numpy(a).cuda(), torch.from_numpy(th).cuda(), transpose).cpu().numpy()
    assert np.array_equal(out, out2)
