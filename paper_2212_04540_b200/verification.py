"""Monte-Carlo verification of the quantizer's statistical guarantees on the
GPU: a port of ``row_mc_statistics``,
``half_fraction_row`` and ``quantizer_verification`` (quantize.py:284-412).

Every draw goes through the production kernel (``kgq_quantize_f32`` on a
block of ``m`` copies of the row, then ``kgq_unpack_codes``), so the counts
are the kernel's own.  The first ``production_trials`` draws are also checked
against the rounding definition on the exported noise of the same keyed
draws (``floor(s) + [u < frac]``, quantize.py:105-113): a mismatch raises
``VerificationError``, as the reference's fast path does (quantize.py:322-328).

Differences from the reference, all statistical-only:
the engine is fp32, so the row is rounded to fp32 before quantization and
the deviations are measured against that fp32 row; R is the fp32 difference
of the fp32 extremes (what the kernel computes); one tensor id per chunk.
"""
import math

import numpy as np
import torch

from .quantize import (RNG_COMPAT, ROUND_STOCHASTIC, QuantConfig, RandomStream, compat_noise_raw53,
                       fast_noise_u16, quantize_tensor, unpack_codes)


class VerificationError(AssertionError):
    """The kernel's counts disagree with the rounding definition (quantize.py:284)."""


def _scaled_fp32(x32: np.ndarray, z32: np.float32, r32: np.float32, bins: int) -> np.ndarray:
    """((x - Z) / R) * B in fp32, the kernel's arithmetic (quantize.py:116-125)."""
    with np.errstate(all="ignore"):
        return ((x32 - z32) / r32) * np.float32(bins)


def row_mc_statistics(row, cfg: QuantConfig, stream: RandomStream, trials: int,
                      production_trials: int = 2000, chunk_rows: int = 1 << 17):
    """quantize.py:288-340: (mean deviation, per-element variance, R, Z) of
    dequantize(quantize(row)) over ``trials`` stochastic draws."""
    if cfg.rounding != ROUND_STOCHASTIC:
        raise ValueError("Monte-Carlo statistics apply to stochastic rounding only")
    if trials < 1:
        raise ValueError("trials must be >= 1")
    x32 = np.asarray(row, dtype=np.float32).reshape(-1)
    d = x32.shape[0]
    z32 = x32.min()
    r32 = np.float32(x32.max() - z32)
    if r32 == 0:
        return np.zeros(d), np.zeros(d), float(r32), float(z32)
    bins = cfg.bins
    scaled = _scaled_fp32(x32, z32, r32, bins)
    floor = np.floor(scaled)
    frac = (scaled - floor).astype(np.float64)
    qcfg = QuantConfig(bits=cfg.bits, rounding=ROUND_STOCHASTIC, group=None, rng=cfg.rng)
    dev = torch.device("cuda")
    xd = torch.from_numpy(x32).to(dev)
    floor_t = torch.from_numpy(floor.astype(np.int64)).to(dev)
    frac_t = torch.from_numpy(frac).to(dev)
    counts = torch.zeros(d, dtype=torch.int64, device=dev)
    done = 0
    while done < trials:
        m = min(chunk_rows, trials - done)
        tid = stream.next_tensor_id()
        q = quantize_tensor(xd.expand(m, d).contiguous(), qcfg, stream, tensor_id=tid)
        codes = unpack_codes(q.codes, cfg.bits, d).to(torch.int64)
        if done < production_trials:
            mp = min(m, production_trials - done)
            if qcfg.rng == RNG_COMPAT:
                u = compat_noise_raw53(stream.seed, tid, mp, d).to(torch.float64) * 2.0 ** -53
            else:
                u = fast_noise_u16(stream.seed, tid, mp, d).to(torch.float64) / 65536.0
            direct = (u < frac_t).sum(0)
            kernel = codes[:mp].sum(0) - mp * floor_t
            if not torch.equal(kernel, direct):
                raise VerificationError("kernel counts diverged from the rounding definition")
            if float(q.ranges[0]) != float(r32) or float(q.offsets[0]) != float(z32):
                raise VerificationError("kernel range/offset differ from the fp32 row extremes")
        counts += codes.sum(0) - m * floor_t
        done += m
    p = counts.cpu().numpy() / trials
    mean_code = floor + p
    x64 = x32.astype(np.float64)
    mean_dev = (np.float64(r32) * mean_code) / bins + np.float64(z32) - x64
    var = (np.float64(r32) / bins) ** 2 * (p * (1.0 - p))
    return mean_dev, var, float(r32), float(z32)


def half_fraction_row(bins: int, dim: int) -> np.ndarray:
    """quantize.py:343-355: scaled interior values with fractional part 1/2
    (Z = 0, R = B by construction)."""
    scaled = np.empty(dim)
    scaled[0] = 0.0
    scaled[-1] = float(bins)
    scaled[1:-1] = (np.arange(dim - 2) % bins) + 0.5
    return scaled


def quantizer_verification(bits_list=(1, 2, 4, 8), n_rows: int = 100, dim: int = 64,
                           trials: int = 100000, seed: int = 0, variance_slack: float = 1.05,
                           tightness_window: float = 0.02, rng: str = "compat") -> dict:
    """quantize.py:358-412: per bit width, (a) per-element |mean dev| <=
    4 sqrt(R^2 / (4 B^2) / trials), (b) per-row variance <= slack * d * R^2 /
    (4 B^2), (c) at half fractions the per-element variance within the window
    of R^2 / (4 B^2).  Rows and stream seeds are derived per width as in the
    reference."""
    if n_rows < 1 or dim < 3 or trials < 1:
        raise ValueError("need n_rows >= 1, dim >= 3 (range anchors plus interior), trials >= 1")
    report = {"trials": trials, "rows": n_rows, "dim": dim, "seed": seed, "rng": rng, "bits": {}}
    all_ok = True
    for bits in bits_list:
        content_rng = np.random.default_rng([seed, bits])
        stream = RandomStream(int(np.random.SeedSequence([seed, bits]).generate_state(1)[0]))
        cfg = QuantConfig(bits=bits, rounding=ROUND_STOCHASTIC, rng=rng)
        bins = cfg.bins
        worst_mean = worst_var = 0.0
        for _ in range(n_rows):
            row = content_rng.uniform(-1.0, 1.0, dim)
            mean_dev, var, r32, _ = row_mc_statistics(row, cfg, stream, trials)
            per_elem = 4.0 * math.sqrt((r32 * r32) / (4.0 * bins * bins) / trials)
            worst_mean = max(worst_mean, float(np.abs(mean_dev).max()) / per_elem)
            worst_var = max(worst_var, float(var.sum()) / (variance_slack * dim * (r32 * r32) / (4.0 * bins * bins)))
        _, tvar, tr32, _ = row_mc_statistics(half_fraction_row(bins, dim), cfg, stream, trials)
        interior = tvar[1:-1] / ((tr32 * tr32) / (4.0 * bins * bins))
        entry = {"bins": bins, "max_mean_dev_over_bound": worst_mean, "max_row_var_over_bound": worst_var,
                 "tightness_min": float(interior.min()), "tightness_max": float(interior.max())}
        entry["passed"] = bool(worst_mean <= 1.0 and worst_var <= 1.0
                               and 1.0 - tightness_window <= entry["tightness_min"]
                               and entry["tightness_max"] <= 1.0 + tightness_window)
        all_ok &= entry["passed"]
        report["bits"][bits] = entry
    report["passed"] = bool(all_ok)
    return report
