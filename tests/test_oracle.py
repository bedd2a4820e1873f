"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py) and published KATs."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import golden_io


def test_philox4x64_random123_kat():
    # Random123 kat_vectors: philox4x64_10, ctr = key = 0
    out = orc.philox4x64_10([0, 0, 0, 0], [0, 0])
    assert [int(v) for v in out] == [0x16554D9ECA36314C, 0xDB20FE9D672D0FDC,
                                     0xD7E772CEE186176B, 0x7E68B68AEC7BA23B]


def test_philox4x32_random123_kat():
    # Random123 kat_vectors: philox4x32_10, ctr = key = 0
    out = orc.philox4x32_10([0, 0, 0, 0], [0, 0])
    assert [int(v) for v in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_philox4x64_matches_numpy_stream():
    z = golden_io.load("philox")
    for i in range(int(z["n_keys"])):
        key = z[f"k{i}_key"]
        raw = z[f"k{i}_raw"]
        for blk in range(4):
            out = orc.philox4x64_10([blk + 1, 0, 0, 0], key)
            assert np.array_equal(out, raw[4 * blk:4 * blk + 4])
        adv = z[f"k{i}_raw_adv1000"]
        for blk in range(2):
            out = orc.philox4x64_10([1000 + blk + 1, 0, 0, 0], key)
            assert np.array_equal(out, adv[4 * blk:4 * blk + 4])


def test_compat_uniforms_match_random_stream():
    z = golden_io.load("philox")
    for i in range(int(z["n_keys"])):
        seed, tid = (int(v) for v in z[f"k{i}_key"])
        ref = z[f"k{i}_matrix_uniforms"]        # RandomStream(seed).matrix_uniforms(tid, 5, 13)
        raw = orc.compat_noise_raw53(seed, tid, 5, 13)
        assert np.array_equal(raw.astype(np.float64) * 2.0 ** -53, ref)


def test_stream_kat_from_survey():
    raw = orc.compat_noise_raw53(0, 0, 1, 4).astype(np.float64) * 2.0 ** -53
    assert raw[0].tolist() == [float.fromhex("0x1.7a5d3204726c0p-7"),
                               float.fromhex("0x1.eeb1585ce5460p-3"),
                               float.fromhex("0x1.c8667a55d9028p-4"),
                               float.fromhex("0x1.20faf40a5fab6p-1")]


@pytest.mark.parametrize("case", list(golden_io.quant_cases()), ids=lambda c: f"c{c['idx']}")
def test_oracle_quantize_matches_reference(case):
    codes, ranges, offsets = orc.quantize(case["x"], case["group"], case["bits"], case["mode"],
                                          case["seed"], case["tid"])
    assert np.array_equal(codes, case["codes"])
    assert np.array_equal(ranges.view(np.uint32), case["ranges"].view(np.uint32))
    assert np.array_equal(offsets.view(np.uint32), case["offsets"].view(np.uint32))
    deq = orc.dequantize(codes, ranges, offsets, case["group"], case["bits"])
    assert np.array_equal(deq.view(np.uint32), case["deq"].reshape(deq.shape).view(np.uint32))


def test_oracle_quantizer_survey_kat_hex():
    cases = {c["bits"]: c for c in golden_io.quant_cases() if c["idx"] < 12 and c["mode"] == 2}
    want = {1: "2400ae", 2: "355d0000aca9", 4: "850fd73600000000f0abc699",
            8: "5588ff007fd56633000000000000000000ffb3a066cc9999"}
    for bits, hx in want.items():
        c = cases[bits]
        codes, ranges, offsets = orc.quantize(c["x"], 8, bits, orc.MODE_SR_COMPAT, 7, 3)
        assert codes.tobytes().hex() == hx
        assert ranges.tolist() == [1.5, 0.0, 5.0]
        assert offsets.tolist() == [-0.5, 1.5, -3.0]


def test_oracle_noise_mode_equals_fast_mode():
    x = np.random.default_rng(3).standard_normal((17, 64)).astype(np.float32)
    u = orc.fast_uniforms(5, 9, 17, 64)
    a = orc.quantize(x, 64, 2, orc.MODE_SR_FAST, 5, 9)
    b = orc.quantize(x, 64, 2, orc.MODE_SR_NOISE, noise=u)
    for p, q in zip(a, b):
        assert np.array_equal(p, q)


def test_oracle_threads_bit_identical():
    x = np.random.default_rng(4).standard_normal((4096, 64)).astype(np.float32)
    for mode in (orc.MODE_SR_COMPAT, orc.MODE_SR_FAST, orc.MODE_NEAREST):
        a = orc.quantize(x, 64, 2, mode, 1, 2, threads=1)
        b = orc.quantize(x, 64, 2, mode, 1, 2, threads=4)
        for p, q in zip(a, b):
            assert np.array_equal(p, q)


def test_oracle_spmm_relu_match_reference():
    z = golden_io.load("spmm")
    for d in (8, 64, 128):
        out = orc.spmm_csr(z["indptr"], z["indices"], z["data"], z[f"e{d}"])
        assert np.array_equal(out.view(np.uint32), z[f"spmm{d}"].view(np.uint32))
        # A_hat is bitwise symmetric, so spmm_t == spmm (test_tape.py:45-50)
        assert np.array_equal(out.view(np.uint32), z[f"spmmt{d}"].view(np.uint32))
        r, m = orc.relu_mask(z[f"e{d}"])
        assert np.array_equal(r, z[f"relu{d}"])
        assert np.array_equal(m, z[f"mask{d}"])


def test_oracle_relu_special_values_match_numpy_maximum():
    """np.maximum(x, 0) (tensorops.py:90): -0.0 -> +0.0, NaN propagated
    (with its sign), inf kept; mask bit x > 0 (NaN -> 0)."""
    x = np.array([[-0.0, 0.0, np.nan, -np.nan, np.inf, -np.inf, -1.0, 2.0,
                   1e-45, -1e-45, 3.0e38, -3.0e38, 0.5, -0.5, np.nan, 7.0]], dtype=np.float32)
    r, m = orc.relu_mask(x)
    ref = np.maximum(x, 0)
    assert np.array_equal(r.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(m, np.packbits((x > 0).reshape(-1), bitorder="little"))


def test_dense_oracle_matches_reference_tape_b32():
    z = golden_io.load("tape")
    for d, layers in ((64, 3), (32, 2)):
        thetas = [z[f"d{d}_theta{i}"] for i in range(layers)]
        loss, grads = orc.dense_step(z[f"d{d}_E0"], thetas, z["indptr"], z["indices"], z["data"],
                                     z["users"], z["pos"], z["neg"], 1e-5, dtype=np.float32)
        pre = f"d{d}_b32_"
        assert loss == pytest.approx(float(z[pre + "loss"]), rel=1e-6)
        for name, g in grads.items():
            np.testing.assert_allclose(g, z[pre + "grad_" + name], rtol=1e-5, atol=1e-7)


def _philox4x32_py(ctr, key, rounds):
    """Random123 Philox4x32 round function restated in plain Python."""
    c0, c1, c2, c3 = (int(v) for v in ctr)
    k0, k1 = (int(v) for v in key)
    m = 0xFFFFFFFF
    for r in range(rounds):
        if r:
            k0, k1 = (k0 + 0x9E3779B9) & m, (k1 + 0xBB67AE85) & m
        p0, p1 = 0xD2511F53 * c0, 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & m, p1 & m, ((p0 >> 32) ^ c3 ^ k1) & m, p0 & m
    return [c0, c1, c2, c3]


def test_fast_stream_is_philox4x32_7():
    """The fast SR stream = Philox4x32 with 7 rounds: the C oracle's
    R-round primitive equals the plain restatement (which at R = 10 reproduces
    the Random123 KAT above), and fast_noise_u16 draws element k of group g
    from call 4(k>>5)+((k>>2)&3), word k&3, half (k>>4)&1."""
    assert orc.FAST_ROUNDS == 7
    assert _philox4x32_py([0, 0, 0, 0], [0, 0], 10) == [int(v) for v in orc.philox4x32_10([0, 0, 0, 0], [0, 0])]
    for ctr, key in (([1, 2, 3, 4], [5, 6]), ([0xFFFFFFFF, 7, 0, 9], [0xDEADBEEF, 0x12345678])):
        assert [int(v) for v in orc.philox4x32(ctr, key, 7)] == _philox4x32_py(ctr, key, 7)
    seed, tid = 0x0123456789ABCDEF, 0xFEDCBA9876543210
    u = orc.fast_noise_u16(seed, tid, 3, 64)
    key = [seed & 0xFFFFFFFF, ((seed >> 32) ^ (tid >> 32)) & 0xFFFFFFFF]
    for g in range(3):
        for k in (0, 5, 17, 33, 63):
            call = 4 * (k >> 5) + ((k >> 2) & 3)
            w = _philox4x32_py([call, g, 0, tid & 0xFFFFFFFF], key, 7)[k & 3]
            assert int(u[g, k]) == (w >> (16 * ((k >> 4) & 1))) & 0xFFFF


@pytest.mark.parametrize("name", ["int", "gauss"])
def test_oracle_evaluate_matches_reference(name):
    """oracle.evaluate (train.py:119-160 restated) == kgact.train.evaluate on
    the fixture (tests/golden/make_eval_golden.py)."""
    z = golden_io.load("eval")
    for k, want in zip(z["ks"], z[f"metrics_{name}"]):
        got = orc.evaluate(int(z["num_users"]), int(z["num_items"]), z["train"], z["test"],
                           z[f"readout_{name}"], int(k))
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)


def test_oracle_topk_stable_order():
    s = np.array([[1.0, 3.0, 3.0, -np.inf, 0.0, -0.0, np.nan, 3.0]])
    assert orc.topk_stable(s, 8)[0].tolist() == [1, 2, 7, 0, 4, 5, 3, 6]


@pytest.mark.parametrize("case", list(golden_io.special_cases()), ids=lambda c: f"s{c['idx']}")
def test_oracle_special_values_match_reference(case):
    """+-0, subnormals, +-inf, NaN (quant_special.npz, written by the reference)."""
    g = case["group"]
    codes, ranges, offsets = orc.quantize(case["x"].reshape(-1, g), g, case["bits"], case["mode"],
                                          case["seed"], case["tid"])
    free = golden_io.mixed_zero_groups(case["x"], g)
    assert np.array_equal(codes, case["codes"])
    assert golden_io.same_bits(ranges, case["ranges"], free)
    assert golden_io.same_bits(offsets, case["offsets"], free)
    deq = orc.dequantize(codes, ranges, offsets, g, case["bits"])
    assert golden_io.same_bits(deq, case["deq"].reshape(deq.shape), free)
