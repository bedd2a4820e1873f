"""Time train.evaluate (Top-K Recall/NDCG on the GPU) on the reference-generated
datasets with a random readout (not a benchmark)."""
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
    evaluate(ds, readout, 20)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = evaluate(ds, readout, 20)
    torch.cuda.synchronize()
    res[name] = {"users": int(len(set(ds.test[:, 0].tolist()))), "items": ds.num_items,
                 "seconds": round(time.perf_counter() - t, 4), "recall_ndcg": r}
print(json.dumps(res))
# split: the top-k kernel alone on one chunk-sized score block
from paper_2212_04540_b200 import functional as F
for name in ("amazon", "lastfm"):
    ds = D.reference_dataset(name)
    s = torch.randn(2048, ds.num_items, device="cuda")
    F.topk_rows(s, 20); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); F.topk_rows(s, 20); b.record(); torch.cuda.synchronize()
    print(json.dumps({name: {"topk_2048_rows_us": round(a.elapsed_time(b) * 1e3, 1),
                             "GBps": round(s.numel() * 4 / a.elapsed_time(b) / 1e6, 1)}}))
