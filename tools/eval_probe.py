"""Time train.evaluate (Top-K Recall/NDCG on the GPU) on the reference-generated
datasets with a random readout, fused (K12) vs the score-block path (cuBLAS +
K11), and check both rank identically on an integer-valued readout (exact
scores).  Not a benchmark."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.train import evaluate

res = {}
for name in ("amazon", "lastfm"):
    ds = D.reference_dataset(name)
    g = torch.Generator(device="cuda").manual_seed(0)
    readout = torch.randn(ds.num_nodes, 64, device="cuda", generator=g)
    readout_int = torch.randint(-3, 4, (ds.num_nodes, 64), device="cuda", generator=g).float()
    row = {"users": int(len(set(ds.test[:, 0].tolist()))), "items": ds.num_items}
    for fused in (True, False):
        evaluate(ds, readout, 20, fused=fused)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            r = evaluate(ds, readout, 20, fused=fused)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        row["fused" if fused else "blocks"] = {"ms": round(1e3 * min(ts), 2), "recall_ndcg": r,
                                               "int_readout": evaluate(ds, readout_int, 20, fused=fused)}
    res[name] = row
print(json.dumps(res))
