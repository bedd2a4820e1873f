"""Trip rate of the reference's criterion 1 (test_acceptance.py:35-79) over
many verification seeds, fast vs compat stream, at the reference's full scale
(100 rows x d=64 x 1e5 draws x b in {1,2,4,8}).

    python tools/verification_seeds.py [n_seeds] [out.json]

A 4-sigma bound over 6,400 elements per width is exceeded by chance on a few
% of (seed, width) cells for ANY unbiased stream; the point of the sweep is
that fast and compat trip at the same rate."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
from paper_2212_04540_b200 import verification as V  # noqa: E402

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 32
out_path = sys.argv[2] if len(sys.argv) > 2 else None
out = {"what": f"quantizer_verification criterion (a) max |mean dev| / 4-sigma bound per width "
               f"(bits 1,2,4,8), full scale (100 rows x d=64 x 1e5 draws), seeds 0..{n_seeds - 1}",
       "seeds": n_seeds}
for rng in ("fast", "compat"):
    vals, t0 = [], time.time()
    for seed in range(n_seeds):
        rep = V.quantizer_verification(bits_list=(1, 2, 4, 8), n_rows=100, dim=64, trials=100000,
                                       seed=seed, rng=rng)
        vals.append([round(rep["bits"][b]["max_mean_dev_over_bound"], 4) for b in (1, 2, 4, 8)])
    cells = [v for row in vals for v in row]
    out[rng] = vals
    out[rng + "_trips"] = sum(v > 1.0 for v in cells)
    out[rng + "_cells"] = len(cells)
    out[rng + "_seeds_failing"] = sum(any(v > 1.0 for v in row) for row in vals)
    out[rng + "_seconds"] = round(time.time() - t0, 1)
out["summary"] = (f"fast: {out['fast_trips']} of {out['fast_cells']} cells over the bound "
                  f"({out['fast_seeds_failing']} of {n_seeds} seeds fail); compat: {out['compat_trips']} of "
                  f"{out['compat_cells']} ({out['compat_seeds_failing']} of {n_seeds} seeds)")
print(json.dumps(out))
if out_path:
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
