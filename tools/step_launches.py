"""Print the kernel sequence of ONE captured training step (graph replay),
Amazon dataset as the reference generates it; run under
ncu --profile-from-start off --metrics gpu__time_duration.sum --csv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.model import ModelConfig, init_params
from paper_2212_04540_b200.train import TrainConfig, AdamState, train_epoch

ds = D.reference_dataset(sys.argv[1] if len(sys.argv) > 1 else "amazon")
adj = D.build_adjacency(ds)
q = kgq.QuantConfig(bits=2, rng="fast")
mcfg, cfg = ModelConfig(layers=3, dim=64, quant=q), TrainConfig(quant=q)
params = init_params(ds.num_nodes, mcfg, 0)
state = AdamState(params.as_dict())
rng, st = np.random.default_rng(0), kgq.RandomStream(0)
train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=6, graphs=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=1, graphs=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
