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
    cfg = kgq.QuantConfig(bits=2, rng="fast")
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
        V.row_mc_statistics(row, kgq.QuantConfig(bits=2, rounding="nearest", rng="fast"), kgq.RandomStream(1), 10)
    # constant row: zero range, zero statistics
    md, v, r0, _ = V.row_mc_statistics(np.full(8, 0.5), cfg, kgq.RandomStream(1), 100)
    assert r0 == 0 and not md.any() and not v.any()


def test_reference_criteria_1_2_full_scale_compat():
    """The reference's acceptance criteria 1-2 (test_acceptance.py:35-91) at
    its own scale and seed: 100 rows x d=64 x 1e5 draws x b in {1,2,4,8},
    VERIFY_SEED = 0, on the reference's stream (rng="compat", the default)."""
    from paper_2212_04540_b200 import verification as V
    rep = V.quantizer_verification(bits_list=(1, 2, 4, 8), n_rows=100, dim=64, trials=100000, seed=0)
    assert rep["rng"] == "compat"
    worst = max(e["max_mean_dev_over_bound"] for e in rep["bits"].values())
    worst_var = max(e["max_row_var_over_bound"] for e in rep["bits"].values())
    tmin = min(e["tightness_min"] for e in rep["bits"].values())
    tmax = max(e["tightness_max"] for e in rep["bits"].values())
    print(f"criterion 1 worst {worst:.3f}x bound; criterion 2 worst {worst_var:.3f}x, "
          f"tightness [{tmin:.4f}, {tmax:.4f}]")
    assert worst <= 1.0                      # criterion 1
    assert worst_var <= 1.0                  # criterion 2 (variance bound)
    assert 0.98 <= tmin and tmax <= 1.02     # criterion 2 (tightness)
