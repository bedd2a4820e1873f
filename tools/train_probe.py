"""Quick GPU training probe on a synthetic shape (not the bench)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.model import ModelConfig, init_params
from paper_2212_04540_b200.train import TrainConfig, AdamState, train_epoch, memory_report

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 2
t0 = time.time()
ds = D.reference_dataset(shape) if shape in D.REFERENCE_DATASETS else D.synth_kg(D.SHAPES[shape], seed=0)
t1 = time.time()
adj = D.build_adjacency(ds)
print(f"gen {t1-t0:.1f}s adj {time.time()-t1:.1f}s nodes {ds.num_nodes} nnz {adj.nnz} train {len(ds.train)} triples {len(ds.triples)}", flush=True)
q = kgq.QuantConfig(bits=bits, rng="fast")
mcfg = ModelConfig(layers=3, dim=64, quant=q)
cfg = TrainConfig(quant=q)
params = init_params(ds.num_nodes, mcfg, 0)
state = AdamState(params.as_dict())
rng = np.random.default_rng(0)
st = kgq.RandomStream(0)
train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=5)
torch.cuda.synchronize()
t = time.time()
s = train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=steps, graphs=len(sys.argv) > 4)
torch.cuda.synchronize()
dt = time.time() - t
print(json.dumps({"ms_per_step": 1e3 * dt / s["steps"], "steps": s["steps"], "loss": s["mean_loss"],
                  "mem": memory_report(s["peak_context_bytes"], s["peak_fp32_equivalent_bytes"], s["adjacency_bytes"])}))
