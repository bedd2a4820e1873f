"""Time eager steps vs captured-graph replays of the training step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data as D, train as T
from paper_2212_04540_b200.model import ModelConfig, init_params

ds = D.synth_kg(D.SHAPES["amazon"], seed=0)
adj = D.build_adjacency(ds)
q = kgq.QuantConfig(bits=2, rng="fast")
mcfg = ModelConfig(layers=3, dim=64, quant=q)
cfg = T.TrainConfig(quant=q)
params = init_params(ds.num_nodes, mcfg, 0)
state = T.AdamState(params.as_dict())
st = kgq.RandomStream(0)
trip = torch.from_numpy(D.sample_negatives(ds, np.random.default_rng(0))).cuda()
for k in range(2):   # warm-up (lazy init must not happen during capture)
    tape, grads, _ = T._record_step(ds, adj, params, mcfg, cfg, st, trip[k * 1024:(k + 1) * 1024], True)
    T.adam_step(params.as_dict(), grads, state, cfg.lr)
torch.cuda.synchronize()
t0 = time.time()
for k in range(5):
    tape, grads, _ = T._record_step(ds, adj, params, mcfg, cfg, st, trip[k * 1024:(k + 1) * 1024], True)
    T.adam_step(params.as_dict(), grads, state, cfg.lr)
torch.cuda.synchronize(); print("eager ms/step", (time.time() - t0) * 1e3 / 5, flush=True)
t0 = time.time()
sg = T._StepGraph(ds, adj, params, mcfg, cfg, state, st, True, 400, "cuda")
torch.cuda.synchronize()
print("capture s", time.time() - t0, flush=True)
for n in (1, 10, 100):
    torch.cuda.synchronize(); t0 = time.time()
    sg.run(trip, 0, n, st, state)
    torch.cuda.synchronize(); print(n, "replays ms/step", (time.time() - t0) * 1e3 / n, flush=True)
torch.cuda.synchronize(); t0 = time.time()
for k in range(20):
    sg.graph.replay()
torch.cuda.synchronize(); print("bare replay ms", (time.time() - t0) * 1e3 / 20)

# the train_epoch graph path, twice (second call reuses the cached capture)
rng = np.random.default_rng(1)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    s = T.train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=300, graphs=True)
    torch.cuda.synchronize(); print("train_epoch graphs ms/step", (time.time() - t0) * 1e3 / s["steps"], flush=True)
torch.cuda.synchronize(); t0 = time.time()
s = T.train_epoch(ds, adj, params, mcfg, cfg, state, st, rng, max_steps=300, graphs=False)
torch.cuda.synchronize(); print("train_epoch eager ms/step", (time.time() - t0) * 1e3 / s["steps"], flush=True)
t0 = time.time(); D.sample_negatives(ds, rng); print("sample_negatives s", time.time() - t0)
