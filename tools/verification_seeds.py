import sys, json
sys.path.insert(0, "/root/repo")
from paper_2212_04540_b200 import verification as V
out = {}
for rng in ("fast", "compat"):
    vals = []
    for seed in range(12):
        rep = V.quantizer_verification(bits_list=(1, 2, 4, 8), n_rows=100, dim=64, trials=100000, seed=seed, rng=rng)
        vals.append([round(rep["bits"][b]["max_mean_dev_over_bound"], 3) for b in (1, 2, 4, 8)])
    out[rng] = vals
print(json.dumps(out))
