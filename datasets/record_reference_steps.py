"""Record step-level fingerprints of the REFERENCE training loop
(kgact.train.train_epoch, train.py:62-103) on a committed reference dataset,
so the GPU run can be pinned step by step, not only after a whole epoch.

Run in the build container (needs /root/reference; CPU, ~2.5 s per Last-FM
step):

    python datasets/record_reference_steps.py lastfm 100

Writes tests/golden/<name>_steps.npz with, for bits 32 and 2 (reference
stream; the GPU side uses rng="compat"):
  * the loss of every step 1..N;
  * after steps 1, 10 and N: the full theta_i, rows ROWS of E0 and a float64
    checksum (sum, sum of |.|) of the whole E0;
  * the step-1 gradients: full theta_i grads and rows ROWS of the E0 grad.
Initialisation follows train_run (train.py:184-187): rng = default_rng(seed),
RandomStream(seed), init_params(num_nodes, model_cfg, seed).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from paper_2212_04540_b200 import data as D  # noqa: E402

CHECKPOINTS = (1, 10)
N_ROWS = 256


def sample_rows(num_nodes: int) -> np.ndarray:
    return np.unique(np.random.default_rng(123).integers(0, num_nodes, N_ROWS)).astype(np.int64)


def run(name, bits, n_steps):
    import kgact.train as KT
    from kgact.data import KgDataset, build_adjacency
    from kgact.model import ModelConfig, init_params
    from kgact.quantize import QuantConfig, RandomStream
    d = D.reference_dataset(name)
    ds = KgDataset(d.num_users, d.num_items, d.num_entities, d.train, d.val, d.test, d.triples,
                   {f"u{u}": u for u in range(d.num_users)}, {f"e{e}": e for e in range(d.num_entities)},
                   {f"r{r}": r for r in range(d.num_relations)})
    q = QuantConfig(bits=bits)
    mcfg = ModelConfig(layers=3, dim=64, quant=q)
    tcfg = KT.TrainConfig(epochs=1, quant=q)
    adj = build_adjacency(ds)
    rng = np.random.default_rng(tcfg.seed)
    stream = RandomStream(tcfg.seed)
    params = init_params(ds.num_nodes, mcfg, tcfg.seed)
    state = KT.AdamState(params.as_dict())
    rows = sample_rows(ds.num_nodes)
    out = {"rows": rows}
    losses = []
    orig_adam, orig_tape = KT.adam_step, KT.Tape

    class RecTape(orig_tape):
        def record_bpr_loss(self, *a, **k):
            w = super().record_bpr_loss(*a, **k)
            losses.append(float(self.loss_value))
            return w

    def rec_adam(param_dict, grads, st, lr):
        if st.step == 0:
            for name_, g in grads.items():
                out[f"grad1_{name_}"] = g[rows] if name_ == "E0" else g.copy()
        orig_adam(param_dict, grads, st, lr)
        if st.step in CHECKPOINTS or st.step == n_steps:
            for name_, p in param_dict.items():
                if name_ == "E0":
                    out[f"s{st.step}_E0_rows"] = p[rows].copy()
                    out[f"s{st.step}_E0_sum"] = np.array([p.astype(np.float64).sum(),
                                                          np.abs(p.astype(np.float64)).sum()])
                else:
                    out[f"s{st.step}_{name_}"] = p.copy()
            print(f"  b{bits} step {st.step}: loss {losses[-1]:.9g}", flush=True)

    KT.adam_step, KT.Tape = rec_adam, RecTape
    try:
        t0 = time.time()
        KT.train_epoch(ds, adj, params, mcfg, tcfg, state, stream, rng, max_steps=n_steps)
    finally:
        KT.adam_step, KT.Tape = orig_adam, orig_tape
    out["losses"] = np.array(losses)
    out["seconds"] = np.array(time.time() - t0)
    return out


def main(name, n_steps):
    res = {"n_steps": np.array(n_steps), "checkpoints": np.array(CHECKPOINTS + (n_steps,))}
    for bits in (32, 2):
        for k, v in run(name, bits, n_steps).items():
            res[f"b{bits}_{k}"] = v
    path = os.path.join(ROOT, "tests", "golden", f"{name}_steps.npz")
    np.savez_compressed(path, **res)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 100)
