"""GPU port of the reference's Monte-Carlo quantizer verification
(quantize.py:284-412): every draw through the production kernel, the first
draws cross-checked against the rounding definition on exported noise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rng", ["fast", "compat"])
def test_quantizer_verification_passes(rng):
    from paper_2212_04540_b200 import verification as V
    rep = V.quantizer_verification(bits_list=(1, 2, 4, 8), n_rows=4, dim=64, trials=40000, seed=0,
                                   rng=rng)
    assert rep["passed"], rep
    for bits, e in rep["bits"].items():
        assert e["max_mean_dev_over_bound"] <= 1.0 and e["max_row_var_over_bound"] <= 1.0


def test_row_mc_statistics_production_check_and_moments():
    import paper_2212_04540_b200 as kgq
    from paper_2212_04540_b200 import verification as V
    cfg = kgq.QuantConfig(bits=2)
    row = np.random.default_rng(3).uniform(-1, 1, 64)
    # production_trials spans several chunks, so the exported-noise check runs per chunk
    mean_dev, var, r, z = V.row_mc_statistics(row, cfg, kgq.RandomStream(9), trials=50000,
                                              production_trials=30000, chunk_rows=10000)
    x32 = row.astype(np.float32)
    assert r == float(np.float32(x32.max() - x32.min())) and z == float(x32.min())
    bound = 4.0 * np.sqrt(r * r / (4 * 9) / 50000)
    assert np.abs(mean_dev).max() <= bound
    assert var.sum() <= 1.05 * 64 * r * r / 36
    # anchors quantize exactly
    assert var[np.argmin(x32)] == 0 and var[np.argmax(x32)] == 0
    with pytest.raises(ValueError):
        V.row_mc_statistics(row, kgq.QuantConfig(bits=2, rounding="nearest"), kgq.RandomStream(1), 10)
    # constant row: zero range, zero statistics
    md, v, r0, _ = V.row_mc_statistics(np.full(8, 0.5), cfg, kgq.RandomStream(1), 100)
    assert r0 == 0 and not md.any() and not v.any()
