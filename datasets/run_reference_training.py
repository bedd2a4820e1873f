"""Train the REFERENCE (kgact.train.train_run, train.py:175-227) on a
committed reference dataset and record its metrics, for bench.py's quality
section and the parity discussion in DESIGN.md.

Run in the build container (needs /root/reference; CPU, ~26 min per epoch at
Amazon shape):

    python datasets/run_reference_training.py amazon BITS EPOCHS
    python datasets/run_reference_training.py amazon --record-json REPORT.json

Merges {"b<BITS>_e<EPOCHS>": {...}} into datasets/<name>_seed0_reference_runs.json.
Quantization config is passed to both ModelConfig and TrainConfig as the
reference CLI does (cli.py:71-75); seed 0, lr 1e-3, batch 1024, l2 1e-5.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from paper_2212_04540_b200 import data as D  # noqa: E402


def record(name, key, rep, wall):
    path = os.path.join(HERE, f"{name}_seed0_reference_runs.json")
    runs = json.load(open(path)) if os.path.exists(path) else {}
    m = rep["metrics"]
    runs[key] = {"epochs": rep["config"]["epochs"], "bits": rep["config"]["bits"],
                 "recall_at_20": m["recall_at_20"], "ndcg_at_20": m["ndcg_at_20"],
                 "loss_curve": rep["loss_curve"], "memory": rep["memory"],
                 "epoch_seconds": rep["timing"]["epoch_seconds"], "wall_s": wall,
                 "host": f"build container, {os.cpu_count()} cores, numpy/scipy (reference as shipped)"}
    with open(path, "w") as f:
        json.dump(runs, f, indent=1, sort_keys=True)


def main(name, bits, epochs):
    from kgact.data import KgDataset
    from kgact.model import ModelConfig
    from kgact.quantize import QuantConfig
    from kgact.train import TrainConfig, train_run
    d = D.reference_dataset(name)
    ds = KgDataset(d.num_users, d.num_items, d.num_entities, d.train, d.val, d.test, d.triples,
                   {f"u{u}": u for u in range(d.num_users)}, {f"e{e}": e for e in range(d.num_entities)},
                   {f"r{r}": r for r in range(d.num_relations)})
    q = QuantConfig(bits=bits)
    t0 = time.time()
    _, rep = train_run(ds, ModelConfig(layers=3, dim=64, quant=q), TrainConfig(epochs=epochs, quant=q))
    record(name, f"b{bits}_e{epochs}", rep, time.time() - t0)
    print(rep["metrics"], rep["memory"])


if __name__ == "__main__":
    if sys.argv[2] == "--record-json":
        # a train_run report the same code path saved as JSON (long runs were
        # started detached): python ... amazon --record-json report.json
        rep = json.load(open(sys.argv[3]))
        record(sys.argv[1], f"b{rep['config']['bits']}_e{rep['config']['epochs']}", rep, rep.get("wall_s", 0.0))
    else:
        main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
