"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports kgact read-only from /root/reference/pkg/src and writes small
``.npz`` files.  Nothing at test/bench time reads /root/reference; the tests
read these committed fixtures instead.

Fixtures:
* philox.npz  -- numpy Philox4x64-10 raw words and RandomStream uniforms
                 (quantize.py:61-102), plus the survey's Random123 KAT.
* quant.npz   -- quantize_tensor / dequantize_tensor outputs
                 (quantize.py:177-210) over a case matrix: bits 1/2/4/8,
                 stochastic (reference stream = "compat"), stochastic fed with
                 our fast-mode noise through a RandomStream subclass (the
                 exported-noise route), and nearest; per-row and per-group
                 (the reference run on x.reshape(-1, G)); edge rows.
* spmm.npz    -- build_adjacency (data.py:230-266) on a tiny synthetic KG,
                 spmm / spmm_t (tensorops.py:37-50), relu + BitMask
                 (tensorops.py:57-92).
* quant_special.npz -- quantize_tensor / dequantize_tensor on rows holding
                 IEEE special values (mixed +-0.0, subnormals, +-inf, NaN,
                 ranges that overflow to inf), G = 64 and 32, all widths and
                 roundings: pins R/Z bits (sign of zero) and the code of a
                 NaN-scaled element (numpy casts NaN to code 0).
* tape.npz    -- Tape forward_all + gathers + BPR (tape.py, model.py) on a
                 toy model: b=32 pass-through and b=2 with fast noise; loss,
                 gradients, packed context codes, ledger counters.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from kgact import quantize as kq  # noqa: E402
from kgact import tensorops as kt  # noqa: E402
from kgact.data import build_adjacency, parse_synth_spec, synth_generate  # noqa: E402
from kgact.model import ModelConfig, forward_all, init_params  # noqa: E402
from kgact.tape import Tape  # noqa: E402

from oracle import oracle as orc  # noqa: E402


class FastNoiseStream(kq.RandomStream):
    """RandomStream whose draws are our fast-mode noise (k/65536, exact in
    float64), keyed per group = per row of the quantized view.  This is the
    exported-noise seam at quantize.py:87-96 consumed at :193."""

    def matrix_uniforms(self, tensor_id, rows, cols, dtype=np.float64):
        return orc.fast_uniforms(self.seed, tensor_id, rows, cols).astype(dtype)


KAT_X = np.array([[0, .3, 1, -.5, .25, .75, .1, -.2],
                  [1.5] * 8,
                  [-3, 2, .5, .125, -1, 1, 0, 1e-3]], dtype=np.float32)


def edge_matrix(rows, cols, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, cols)).astype(np.float32)
    x[::7] = x[::7, :1]                    # constant rows (R == 0)
    x[3::5] *= np.float32(1e-30)           # tiny-range rows
    x[2::9] = np.abs(x[2::9])              # rows with min near 0 ...
    x[2::9, ::3] = 0.0                     # ... and exact zeros (post-ReLU like)
    x[4::11] = -np.abs(x[4::11]) - 5.0     # all-negative rows
    x[6::13, 1::2] = x[6::13, :1]          # repeated min/max values
    return x


def quant_cases():
    cases = []
    # survey KAT: RandomStream(7), tid 3
    for bits in (1, 2, 4, 8):
        cases.append(dict(x=KAT_X, group=8, bits=bits, mode="compat", seed=7, tid=3))
        cases.append(dict(x=KAT_X, group=8, bits=bits, mode="nearest", seed=0, tid=0))
        cases.append(dict(x=KAT_X, group=8, bits=bits, mode="fast", seed=7, tid=3))
    shapes = [(37, 13), (50, 64), (33, 128), (20, 256), (10, 3), (64, 32), (9, 96)]
    for si, (r, c) in enumerate(shapes):
        x = edge_matrix(r, c, 100 + si)
        for bits in (1, 2, 4, 8):
            for mode in ("compat", "fast", "nearest"):
                cases.append(dict(x=x, group=c, bits=bits, mode=mode, seed=11 + si,
                                  tid=5 + bits))
    # per-group quantization: the reference run on x.reshape(-1, G)
    for (r, c, g) in [(16, 256, 64), (8, 128, 64), (12, 256, 128), (6, 512, 256)]:
        x = edge_matrix(r, c, 7 * r + c)
        for bits in (2, 4, 8):
            for mode in ("compat", "fast", "nearest"):
                cases.append(dict(x=x, group=g, bits=bits, mode=mode, seed=3, tid=2**40 + bits))
    # big seeds / tensor ids (64-bit keys)
    x = edge_matrix(40, 64, 999)
    cases.append(dict(x=x, group=64, bits=2, mode="compat", seed=2**64 - 1, tid=2**63 + 5))
    cases.append(dict(x=x, group=64, bits=2, mode="fast", seed=2**64 - 1, tid=2**63 + 5))
    return cases


def special_matrix(seed=0):
    """64-column rows of IEEE special values (quantize.py:184-186 min/max,
    :116-125 scaling, :128-132 rounding, :199-210 dequantize)."""
    rng = np.random.default_rng(seed)
    f = np.float32
    rows = []
    base = lambda: rng.standard_normal(64).astype(f)            # noqa: E731
    z = np.zeros(64, f)
    r = z.copy(); r[1::3] = -0.0; rows.append(r)                # mixed +0/-0 (min sign: numpy SIMD order)
    rows.append(np.full(64, -0.0, f))                           # all -0
    rows.append(np.zeros(64, f))                                # all +0
    r = np.abs(base()); r[::4] = -0.0; rows.append(r)           # -0 min with positives (post-ReLU-like)
    r = np.abs(base()); r[::4] = 0.0; rows.append(r)            # +0 min with positives
    r = -np.abs(base()); r[::5] = -0.0; rows.append(r)          # -0 max with negatives
    rows.append((base() * f(1e-39)).astype(f))                  # subnormal values only
    r = (np.abs(base()) * f(1e-40)).astype(f); r[::3] = 0.0; rows.append(r)   # subnormals + zeros
    r = base(); r[7] = f(1e-41); rows.append(r)                 # one subnormal among normals
    r = (base() * f(1e-37)).astype(f); rows.append(r)           # near the normal boundary
    rows.append(np.full(64, f(1.4e-45)))                        # constant min-subnormal
    r = base(); r[5] = np.inf; rows.append(r)                   # +inf -> R = inf
    r = base(); r[9] = -np.inf; rows.append(r)                  # -inf -> Z = -inf
    r = base(); r[2] = np.inf; r[3] = -np.inf; rows.append(r)   # both -> R = inf
    rows.append(np.full(64, np.inf, f))                         # all +inf (R = nan)
    rows.append(np.full(64, -np.inf, f))                        # all -inf
    r = base(); r[0] = f(3e38); r[1] = f(-3e38); rows.append(r)  # range overflows to inf
    r = base(); r[63] = f(3.4e38); rows.append(r)               # huge max, finite range
    r = base(); r[11] = np.nan; rows.append(r)                  # NaN -> R = Z = nan
    rows.append(np.full(64, f(-7.25)))                          # constant negative
    for _ in range(4):
        rows.append(base())                                     # plain rows around them
    return np.stack(rows).astype(f)


SPECIAL_NAN_ROWS = (18,)   # rows whose R/Z are NaN (payload is platform-defined)


def special_cases():
    x = special_matrix()
    cases = []
    for g in (64, 32):
        for bits in (1, 2, 4, 8):
            for mode in ("compat", "fast", "nearest"):
                cases.append(dict(x=x, group=g, bits=bits, mode=mode, seed=31 + g, tid=bits))
    return cases


def make_special():
    import warnings
    out = {}
    cases = special_cases()
    for i, cs in enumerate(cases):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")   # numpy warns on inf-inf, inf/inf and NaN casts
            q, deq = run_quant_case(cs)
        p = f"c{i}_"
        out[p + "x"] = cs["x"]
        out[p + "meta"] = np.array([cs["group"], cs["bits"],
                                    {"nearest": 0, "fast": 1, "compat": 2}[cs["mode"]]],
                                   dtype=np.int64)
        out[p + "seed_tid"] = np.array([cs["seed"], cs["tid"]], dtype=np.uint64)
        out[p + "codes"] = q.codes
        out[p + "ranges"] = q.ranges
        out[p + "offsets"] = q.offsets
        out[p + "deq"] = deq
        out[p + "stored_bytes"] = np.array(kq.stored_bytes(q))
    out["n_cases"] = np.array(len(cases))
    return out


def run_quant_case(cs):
    x = cs["x"].reshape(-1, cs["group"])
    cfg = kq.QuantConfig(bits=cs["bits"],
                         rounding="nearest" if cs["mode"] == "nearest" else "stochastic")
    if cs["mode"] == "compat":
        stream = kq.RandomStream(cs["seed"])
    elif cs["mode"] == "fast":
        stream = FastNoiseStream(cs["seed"])
    else:
        stream = None
    q = kq.quantize_tensor(x, cfg, stream, tensor_id=cs["tid"] if stream else None)
    deq = kq.dequantize_tensor(q, np.float32)
    return q, deq


def make_philox():
    from numpy.random import Generator, Philox
    out = {}
    keys = [(0, 0), (7, 3), (2**64 - 1, 5), (123456789, 2**63 + 5)]
    for i, (s, t) in enumerate(keys):
        bg = Philox(key=np.array([s, t], dtype=np.uint64))
        out[f"k{i}_key"] = np.array([s, t], dtype=np.uint64)
        out[f"k{i}_raw"] = bg.random_raw(16).astype(np.uint64)
        bg2 = Philox(key=np.array([s, t], dtype=np.uint64))
        bg2.advance(1000)
        out[f"k{i}_raw_adv1000"] = bg2.random_raw(8).astype(np.uint64)
        st = kq.RandomStream(s)
        out[f"k{i}_matrix_uniforms"] = st.matrix_uniforms(t, 5, 13)
    out["n_keys"] = np.array(len(keys))
    return out


def make_quant():
    out = {}
    cases = quant_cases()
    for i, cs in enumerate(cases):
        q, deq = run_quant_case(cs)
        p = f"c{i}_"
        out[p + "x"] = cs["x"]
        out[p + "meta"] = np.array([cs["group"], cs["bits"],
                                    {"nearest": 0, "fast": 1, "compat": 2}[cs["mode"]]],
                                   dtype=np.int64)
        out[p + "seed_tid"] = np.array([cs["seed"], cs["tid"]], dtype=np.uint64)
        out[p + "codes"] = q.codes
        out[p + "ranges"] = q.ranges
        out[p + "offsets"] = q.offsets
        out[p + "deq"] = deq
        out[p + "stored_bytes"] = np.array(kq.stored_bytes(q))
    out["n_cases"] = np.array(len(cases))
    # packing known answers (test_quantize.py:131-135)
    out["pack_1"] = kq.pack_bits([1, 0, 1, 1, 0, 0, 0, 0], 1)
    out["pack_2"] = kq.pack_bits([3, 2, 1, 0], 2)
    return out


def tiny_kg():
    spec = parse_synth_spec("default,users=60,items=40,entities=120,relations=4,groups=4")
    return synth_generate(spec, seed=0)


def make_spmm():
    ds = tiny_kg()
    adj = build_adjacency(ds)
    rng = np.random.default_rng(5)
    out = {"indptr": adj.indptr.astype(np.int32), "indices": adj.indices.astype(np.int32),
           "data": adj.data.astype(np.float32), "n": np.array(adj.shape[0])}
    for d in (8, 64, 128):
        e = rng.standard_normal((adj.shape[0], d)).astype(np.float32)
        out[f"e{d}"] = e
        out[f"spmm{d}"] = kt.spmm(adj, e)
        out[f"spmmt{d}"] = kt.spmm_t(adj, e)
        relu_out, mask = kt.relu(e)
        out[f"relu{d}"] = relu_out
        out[f"mask{d}"] = mask.packed
    # the survey's 60-shape ordered-accumulation sweep, in miniature
    return out


def make_tape():
    ds = tiny_kg()
    adj = build_adjacency(ds)
    out = {"indptr": adj.indptr.astype(np.int32), "indices": adj.indices.astype(np.int32),
           "data": adj.data.astype(np.float32), "n": np.array(adj.shape[0])}
    rng = np.random.default_rng(9)
    batch = 48
    users = rng.integers(0, ds.num_users, batch).astype(np.int32)
    pos = (ds.num_users + rng.integers(0, ds.num_items, batch)).astype(np.int32)
    neg = (ds.num_users + rng.integers(0, ds.num_items, batch)).astype(np.int32)
    out.update(users=users, pos=pos, neg=neg)
    for d, layers in ((64, 3), (32, 2)):
        mcfg = ModelConfig(layers=layers, dim=d)
        params = init_params(adj.shape[0], mcfg, seed=1)
        out[f"d{d}_E0"] = params.entity_embeddings
        for i, w in enumerate(params.layer_weights):
            out[f"d{d}_theta{i}"] = w
        for bits, stream_cls in ((32, kq.RandomStream), (2, FastNoiseStream), (4, FastNoiseStream),
                                 (8, FastNoiseStream)):
            seed = 21
            stream = stream_cls(seed)
            cfg = kq.QuantConfig(bits=bits)
            tape = Tape(cfg, stream)
            readout = forward_all(tape, params, adj, ModelConfig(layers=layers, dim=d, quant=cfg))
            u = tape.record_gather(readout, users)
            p = tape.record_gather(readout, pos)
            n = tape.record_gather(readout, neg)
            tape.record_bpr_loss(u, p, n, 1e-5)
            pre = f"d{d}_b{bits}_"
            out[pre + "readout"] = readout.value
            # the packed quantized contexts, in tape order (tids 0..L+2)
            qs = []
            for node in tape.nodes:
                if node.kind == "mm":
                    qs.append(node.context["q"])
                if node.kind == "bpr_loss":
                    qs += [node.context["qu"], node.context["qp"], node.context["qn"]]
            for k, q in enumerate(qs):
                if bits != 32:
                    out[pre + f"q{k}_codes"] = q.codes
                    out[pre + f"q{k}_ranges"] = q.ranges
                    out[pre + f"q{k}_offsets"] = q.offsets
            out[pre + "peak_ctx"] = np.array(tape.peak_context_bytes)
            out[pre + "peak_eq"] = np.array(tape.peak_fp32_equiv_bytes)
            grads = tape.backward()
            out[pre + "loss"] = np.array(tape.loss_value)
            for name, g in grads.items():
                out[pre + "grad_" + name] = g
            out[pre + "retained"] = np.array(tape.current_context_bytes)
            out[pre + "n_tids"] = np.array(stream._next_tensor_id)
    return out


C1_SPEC = "default,users=2000,items=3000,entities=10000,relations=20"


def make_c1():
    """BASELINE configs[0]: the reference's own dataset,
    adjacency, first-epoch batches and short training runs (b=32 and b=2 fed
    the fast-mode noise) -- the Recall@20 parity target."""
    from kgact import train as ktrain
    from kgact.data import sample_negatives
    ds = synth_generate(parse_synth_spec(C1_SPEC), seed=0)
    adj = build_adjacency(ds)
    out = {"num_users": np.array(ds.num_users), "num_items": np.array(ds.num_items),
           "num_entities": np.array(ds.num_entities), "num_relations": np.array(len(ds.relation_vocab)),
           "train": ds.train, "val": ds.val, "test": ds.test, "triples": ds.triples,
           "adj_indptr": adj.indptr.astype(np.int32), "adj_indices": adj.indices.astype(np.int32),
           "adj_data": adj.data.astype(np.float32)}
    rng = np.random.default_rng(0)
    trip = sample_negatives(ds, rng)
    order = rng.permutation(len(trip))
    out["epoch0_triples"] = trip[order]
    epochs = 3
    for bits in (32, 2):
        mcfg = ModelConfig(layers=2, dim=64, quant=kq.QuantConfig(bits=bits))
        tcfg = ktrain.TrainConfig(epochs=epochs, batch_size=1024, seed=0,
                                  quant=kq.QuantConfig(bits=bits))
        saved = ktrain.RandomStream
        ktrain.RandomStream = FastNoiseStream
        try:
            _, rep = ktrain.train_run(ds, mcfg, tcfg, adjacency=adj)
        finally:
            ktrain.RandomStream = saved
        pre = f"run_b{bits}_"
        out[pre + "loss_curve"] = np.array(rep["loss_curve"])
        out[pre + "recall"] = np.array(rep["metrics"]["recall_at_20"])
        out[pre + "ndcg"] = np.array(rep["metrics"]["ndcg_at_20"])
        out[pre + "peak_ctx"] = np.array(rep["memory"]["activation_bytes_peak"])
        out[pre + "peak_eq"] = np.array(rep["memory"]["fp32_equivalent_bytes"])
        out[pre + "epoch_seconds"] = np.array(rep["timing"]["epoch_seconds"])
    out["run_epochs"] = np.array(epochs)
    return out


def main():
    if sys.argv[1:] == ["special"]:
        np.savez_compressed(os.path.join(HERE, "quant_special.npz"), **make_special())
        return
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **make_c1())
    np.savez_compressed(os.path.join(HERE, "philox.npz"), **make_philox())
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **make_quant())
    np.savez_compressed(os.path.join(HERE, "quant_special.npz"), **make_special())
    np.savez_compressed(os.path.join(HERE, "spmm.npz"), **make_spmm())
    np.savez_compressed(os.path.join(HERE, "tape.npz"), **make_tape())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
