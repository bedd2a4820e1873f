"""Training quality vs SR noise stream (not a benchmark): one Last-FM epoch
from the reference's initial state and batches, INT2, with the noise stream
seed varied (params / batches fixed): fast vs compat."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.model import ModelConfig, init_params, embed
from paper_2212_04540_b200.train import AdamState, TrainConfig, evaluate, train_epoch

shape = sys.argv[1] if len(sys.argv) > 1 else "lastfm"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast", "compat"]
seeds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2]
ds = D.reference_dataset(shape)
adj = D.build_adjacency(ds)
out = {}
for mode in modes:
    for s in seeds:
        bits = 32 if mode == "fp32" else 2
        q = kgq.QuantConfig(bits=bits, rng="fast" if mode == "fp32" else mode)
        mcfg, cfg = ModelConfig(layers=3, dim=64, quant=q), TrainConfig(quant=q)
        params = init_params(ds.num_nodes, mcfg, 0)
        state = AdamState(params.as_dict())
        st = train_epoch(ds, adj, params, mcfg, cfg, state, kgq.RandomStream(1000 + s), np.random.default_rng(0),
                         graphs=True)
        r, n = evaluate(ds, embed(params, adj, mcfg), 20)
        out[f"{mode}_s{s}"] = [round(r, 5), round(n, 5), round(st["mean_loss"], 6)]
        print(mode, s, out[f"{mode}_s{s}"], flush=True)
print(json.dumps(out))
