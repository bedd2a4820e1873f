import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.model import ModelConfig, init_params, embed
from paper_2212_04540_b200.train import AdamState, TrainConfig, evaluate, train_epoch
for shape in ("amazon", "lastfm"):
    ds = D.reference_dataset(shape); adj = D.build_adjacency(ds)
    for fused in (True, False):
        q = kgq.QuantConfig(bits=32, rng="fast")
        mcfg, cfg = ModelConfig(layers=3, dim=64, quant=q), TrainConfig(quant=q)
        params = init_params(ds.num_nodes, mcfg, 0); state = AdamState(params.as_dict())
        st = train_epoch(ds, adj, params, mcfg, cfg, state, kgq.RandomStream(0), np.random.default_rng(0), fused=fused, graphs=True)
        r, n = evaluate(ds, embed(params, adj, mcfg), 20)
        print(shape, "fused" if fused else "unfused", round(st["mean_loss"], 7), round(r, 5), round(n, 5), flush=True)
