"""torch.profiler breakdown of train.evaluate on the Amazon dataset (not a benchmark)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.train import evaluate

ds = D.reference_dataset("amazon")
readout = torch.randn(ds.num_nodes, 64, device="cuda")
evaluate(ds, readout, 20)
torch.cuda.synchronize()
t = time.perf_counter()
evaluate(ds, readout, 20)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as p:
    evaluate(ds, readout, 20)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="self_cpu_time_total", row_limit=15))
print(p.key_averages().table(sort_by="self_cuda_time_total", row_limit=10))
