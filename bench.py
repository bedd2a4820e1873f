#!/usr/bin/env python
"""Benchmark: quantize+dequantize HBM GB/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the largest single-GPU microbench shape):
fp32 activations 64M x 128 (32 GB, far larger than the 126 MB L2, so no L2
flush is needed), INT2, group 64, stochastic rounding with the fast
Philox4x32-7 noise.  One step = one fused quantize+pack (K1) plus one
unpack+dequantize (K2) pass over the whole tensor through the public API.

Bytes are algorithmic: per element 4 (fp32) + b/8 (codes)
+ 8/G (fp32 range and offset per group), counted once for K1 and once for K2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun every rank quantizes its own 64M x 128 shard (row offset =
rank * rows, so the noise keys are global): weak scaling, no collective on
the data path.  ``--impl reference`` times the CPU port of the reference
algorithm (oracle/, compat Philox4x64 stream) on the host cores.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quantize+dequantize HBM GB/s (%peak); KGAT epoch/s and activation MB at INT2"
UNIT = "GB/s"


def algo_bytes_per_elem(bits, group):
    return 4.0 + bits / 8.0 + 8.0 / group


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or getattr(args, "partitioned", False):
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29000 + os.getpid() % 1000))
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_port_run(rows, cols, bits, group, threads, seed=1, tid=0, min_seconds=0.0, max_reps=1, rng="compat"):
    """The oracle port of the reference quantize/dequantize on host cores, with
    the reference's numpy Philox4x64-10 stream (rng="compat") or the fast
    stream the GPU arm's headline uses (rng="fast": the reference's rounding
    fed that noise, the exported-noise route).  Returns (GB/s, seconds, reps)."""
    from oracle import oracle as orc
    mode = orc.MODE_SR_COMPAT if rng == "compat" else orc.MODE_SR_FAST
    x = np.random.default_rng(0).standard_normal((rows * cols // group, group), dtype=np.float32)
    orc.lib()
    t0 = time.perf_counter()
    reps = 0
    while True:
        c, r, o = orc.quantize(x, group, bits, mode, seed, tid + reps, threads=threads)
        orc.dequantize(c, r, o, group, bits, threads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if reps >= max_reps or (el >= min_seconds and reps >= 1):
            break
    el = time.perf_counter() - t0
    gb = 2 * rows * cols * algo_bytes_per_elem(bits, group) * reps / 1e9
    return gb / el, el, reps


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    rows = args.ref_rows
    # the GPU arm's config, unchanged: same workload, widths, group and noise
    # stream (the per-element CPU rate does not depend on the row count, so
    # each step is a bounded row sample, stated in cpu_baseline.sample)
    cfg = workload_config(args)
    sample = f"{rows}x{args.cols} fp32 rows per step (bounded sample of the {args.rows}-row workload)"
    for _ in range(args.warmup):
        cpu_port_run(rows, args.cols, args.bits, args.group, threads, rng=args.rng)
    times = []
    for s in range(args.steps):
        gbs, el, _ = cpu_port_run(rows, args.cols, args.bits, args.group, threads, tid=1000 + s, rng=args.rng)
        times.append(el)
    total_gb = 2 * rows * args.cols * algo_bytes_per_elem(args.bits, args.group) * args.steps / 1e9
    value = total_gb / sum(times)
    # beside it: the reference's own numpy Philox4x64-10 stream (rng="compat")
    other = "compat" if args.rng != "compat" else "fast"
    o_gbs, _, _ = cpu_port_run(rows, args.cols, args.bits, args.group, threads, tid=2000, rng=other)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample + f"; oracle/kgq_oracle.c restatement of quantize_tensor/"
                         f"dequantize_tensor (quantize.py:177-210), rng={args.rng} as in config, "
                         "pthreads over groups",
                         f"value_rng_{other}": round(o_gbs, 4)},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def pcie_probe(h_in, h_out):
    """Host<->device copy ceilings on the e2e leg's own pinned buffers, CUDA
    events: H2D alone, D2H alone, and both directions at once on two streams
    (the e2e step's traffic pattern).  GB/s per direction."""
    import torch
    n = h_in.numel()
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.empty(n, dtype=torch.float32, device="cuda")
    hi, ho = h_in.view(-1), h_out.view(-1)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        # best of `reps` single runs: a PCIe link's throughput varies from run
        # to run (other tenants of the switch, IOMMU), the ceiling is the best
        fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 1e3)
        return best

    def both():
        # H2D and D2H at once, in the e2e pipeline's 16 chunks per direction
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        s1.wait_event(ev)
        s2.wait_event(ev)
        step = (n + 15) // 16
        for lo in range(0, n, step):
            hi_ = min(n, lo + step)
            with torch.cuda.stream(s1):
                d_in[lo:hi_].copy_(hi[lo:hi_], non_blocking=True)
            with torch.cuda.stream(s2):
                ho[lo:hi_].copy_(d_out[lo:hi_], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    gb = n * 4 / 1e9
    h2d = gb / timed(lambda: d_in.copy_(hi, non_blocking=True))
    d2h = gb / timed(lambda: ho.copy_(d_out, non_blocking=True))
    t_both = timed(both)
    del d_in, d_out
    return {"h2d_GBps": round(h2d, 2), "d2h_GBps": round(d2h, 2),
            "both_h2d_GBps": round(gb / t_both, 2), "both_d2h_GBps": round(gb / t_both, 2),
            "bytes_each_way": int(n * 4),
            "note": "pinned copies of the e2e buffers; 'both' = H2D and D2H on two streams at once"}


def workload_config(args):
    return {"workload": f"quantize+dequantize microbench (configs[1]) {args.rows}x{args.cols} fp32, "
                        f"INT{args.bits}, group {args.group}, SR rng={args.rng}",
            "rows_per_gpu": args.rows, "cols": args.cols, "bits": args.bits, "group": args.group,
            "rounding": "stochastic", "rng": args.rng,
            "l2": "inputs (%.1f GB/GPU) larger than the 126 MB L2; no flush needed"
                  % (args.rows * args.cols * 4 / 1e9)}


def train_bench(args, world, rank, shape=None, with_fp32=True, with_cpu=True):
    """KGNN training on the Amazon-book-shaped synthetic KG (BASELINE configs[3];
    159,251 nodes, 3 layers, d=64, B=1024) at INT2: ms/step, epochs/s and the
    activation ledger.  world > 1: row-partitioned step (parallel.py, NCCL)."""
    import torch
    import paper_2212_04540_b200 as kgq
    from paper_2212_04540_b200 import data as D
    from paper_2212_04540_b200.model import ModelConfig, init_params
    from paper_2212_04540_b200.train import AdamState, TrainConfig, adam_step, memory_report, train_epoch

    shape = shape or args.train_shape
    if shape in D.REFERENCE_DATASETS:
        ds = D.reference_dataset(shape)
        origin = "reference generator (synth_generate seed 0, datasets/)"
    else:
        ds = D.synth_kg(D.SHAPES[shape], seed=0)
        origin = "vectorized generator"
    steps_per_epoch = (len(ds.train) + 1023) // 1024
    out = {"workload": f"{shape}-shaped synthetic KG from the {origin}: {ds.num_users} users, "
                       f"{ds.num_items} items, {ds.num_entities} entities, {len(ds.triples)} triples, "
                       f"{len(ds.train)} train pairs; KGNN 3 layers d=64, batch 1024, INT2 stochastic (fast rng)",
           "steps_per_epoch": steps_per_epoch, "n_gpus": world}
    res, hbm_peak = {}, {}
    for bits in ((2, 4, 32) if with_fp32 else (2,)):
        q = kgq.QuantConfig(bits=bits, rng="fast")
        mcfg = ModelConfig(layers=3, dim=64, quant=q)
        cfg = TrainConfig(quant=q)
        rng = np.random.default_rng(0)
        stream = kgq.RandomStream(0)
        cur = torch.cuda.current_stream()
        if world == 1 and not args.partitioned:
            adj = D.build_adjacency(ds)
            params = init_params(ds.num_nodes, mcfg, 0)
            state = AdamState(params.as_dict())
            # warm-up: eager steps, then (graphs) one full epoch that captures
            # the step graph at full-epoch capacity (capture not timed)
            train_epoch(ds, adj, params, mcfg, cfg, state, stream, rng, max_steps=args.warmup + 2)
            graphs = not args.no_graphs
            if graphs:
                train_epoch(ds, adj, params, mcfg, cfg, state, stream, rng, graphs=True)
            # (1) step time: K steps of the hot path on batches already on the
            #     device (the epoch's negatives are sampled on the host first,
            #     outside the timed region), CUDA events on the launch stream
            trip = torch.from_numpy(D.sample_negatives(ds, np.random.default_rng(1))).cuda()
            k = min(args.train_steps, len(trip) // 1024)
            # (0) HBM a step allocates beyond the resident state (params, Adam
            #     moments, adjacency, batches): one eager step under
            #     torch.cuda.max_memory_allocated (graph replays reuse a pool)
            from paper_2212_04540_b200.train import _record_step
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            base_alloc = torch.cuda.memory_allocated()
            _, g0, _ = _record_step(ds, adj, params, mcfg, cfg, stream, trip[:1024], True)
            del g0
            torch.cuda.synchronize()
            step_peak = torch.cuda.max_memory_allocated() - base_alloc
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if graphs:
                from paper_2212_04540_b200 import train as T
                sg = next(iter(T._GRAPHS.values()))
                sg.run(trip, 0, 2, stream, state)            # warm replays
                torch.cuda.synchronize()
                a.record(cur)
                sg.run(trip, 0, k, stream, state)
                b.record(cur)
            else:
                from paper_2212_04540_b200.train import _record_step, adam_step
                a.record(cur)
                for i in range(k):
                    _, grads, _ = _record_step(ds, adj, params, mcfg, cfg, stream, trip[i * 1024:(i + 1) * 1024],
                                               True)
                    adam_step(params.as_dict(), grads, state, cfg.lr)
                b.record(cur)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / k
            # (2) epochs as a user runs them (train_run, train.py:175-227): 3
            #     full epochs from scratch, negatives drawn on a host thread one
            #     epoch ahead; epoch time = median of epochs >= 2 (the
            #     reference's convention), wall clock
            from paper_2212_04540_b200.train import train_run
            _, rep = train_run(ds, mcfg, replace(cfg, epochs=3), adjacency=adj, graphs=graphs)
            epoch_s = float(np.median(rep["timing"]["epoch_seconds"][1:]))
            m = rep["memory"]
            mem = memory_report(m["activation_bytes_peak"], m["fp32_equivalent_bytes"], m.get("adjacency_bytes", 0))
            res[bits] = (ms, mem, rep["loss_curve"][-1], epoch_s)
            hbm_peak[bits] = step_peak
        else:
            ms = _partitioned_train_ms(ds, mcfg, cfg, stream, rng, world, rank, args)
            res[bits] = (ms, None, None, None)
    ms2, mem2, loss2, ep2 = res[2]
    if ep2 is None:      # partitioned: extrapolated from the step time
        ep2 = ms2 * steps_per_epoch / 1e3
        out["epoch_note"] = "epoch_s = ms_per_step x steps_per_epoch (partitioned path)"
    else:
        out["epoch_note"] = ("epoch_s measured: median of epochs 2-3 of a 3-epoch train_run (every batch, "
                             "host negative sampling one epoch ahead on a thread), wall clock; ms_per_step: "
                             "device time of the captured step on device-resident batches, CUDA events")
    out.update({"ms_per_step": round(ms2, 3), "epoch_s": round(ep2, 3),
                "epochs_per_s": round(1.0 / ep2, 4), "timed_steps": args.train_steps})
    if with_fp32:
        ms32 = res[32][0]
        out.update({"fp32_ms_per_step": round(ms32, 3), "int2_time_overhead_vs_fp32": round(ms2 / ms32 - 1.0, 4)})
    if 4 in res:
        ms4, mem4, _, ep4 = res[4]
        out["int4"] = {"ms_per_step": round(ms4, 3)}
        if ep4 is not None:
            out["int4"]["epoch_s"] = round(ep4, 3)
        if mem4 is not None:
            out["int4"]["activation_MB_incl_adjacency"] = round(mem4["activation_bytes_peak"] / 1e6, 3)
            out["int4"]["activation_MB_excl_adjacency"] = round(mem4["activation_bytes_excl_adjacency"] / 1e6, 3)
            out["int4"]["ratio_excl_adjacency"] = round(mem4["compression_ratio_excl_adjacency"], 3)
    if world == 1 and rank == 0 and not args.skip_cpu and with_cpu:
        # CPU port of the reference step (oracle/oracle.py dense engine: scipy
        # CSR spmm + numpy GEMMs, the reference's op structure), 2 steps
        from oracle import oracle as orc
        indptr, indices, vals = D.adjacency_arrays(ds)
        p0 = init_params(ds.num_nodes, ModelConfig(layers=3, dim=64), 0, device="cpu")
        e0 = p0.entity_embeddings.numpy()
        ths = [t.numpy() for t in p0.layer_weights]
        trip = D.sample_negatives(ds, np.random.default_rng(0))[:1024]
        t0 = time.perf_counter()
        for _ in range(2):
            orc.dense_step(e0, ths, indptr, indices, vals, trip[:, 0], ds.num_users + trip[:, 1],
                           ds.num_users + trip[:, 2], 1e-5, dtype=np.float32)
        cs = (time.perf_counter() - t0) / 2
        out["cpu_baseline"] = {"value": round(cs * 1e3, 1), "unit": "ms/step", "cores": os.cpu_count(),
                               "kind": "port",
                               "sample": "2 fp32 steps of oracle.dense_step (numpy/scipy restatement of "
                                         "the reference Tape step, no quantization) on the same graph"}
    if world == 1 and shape in ("amazon", "lastfm"):
        # the step's dominant kernel (K4 SpMM, ~60 % of the step): its L2
        # random-row gather rate against the ceiling measured by
        # tools/tc_probe/l2_gather.cu on this pool (profiles/r1_l2_gather_ceiling.json)
        from paper_2212_04540_b200 import tensorops as TO
        adj = D.build_adjacency(ds)
        x = torch.randn(ds.num_nodes, 64, device="cuda")
        TO.spmm(adj, x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for _ in range(20):
            TO.spmm(adj, x)
        b.record(cur)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        gbs = adj.nnz * (64 * 4 + 8) / us / 1e3
        ceil_path = os.path.join(ROOT, "profiles", "r1_l2_gather_ceiling.json")
        ceiling = json.load(open(ceil_path))["GBps"] if os.path.exists(ceil_path) else None
        out["roofline_spmm"] = {"kernel": "spmm_kernel (K4, bit-exact ordered CSR SpMM)", "bound": "l2-gather",
                                "us": round(us, 1), "achieved": round(gbs, 1), "unit": "GB/s",
                                "peak": ceiling, "frac": round(gbs / ceiling, 4) if ceiling else None,
                                "peak_source": "measured L2 random-row gather ceiling (tools/tc_probe/l2_gather.cu)",
                                "bytes_per_nnz": 64 * 4 + 8}
        del x
    if mem2 is not None:
        mb = lambda v: round(v / 1e6, 3)
        out["activation_MB"] = {
            "int2_incl_adjacency": mb(mem2["activation_bytes_peak"]),
            "fp32_incl_adjacency": mb(mem2["fp32_equivalent_bytes"]),
            "ratio_incl_adjacency": round(mem2["compression_ratio"], 3),
            "int2_excl_adjacency": mb(mem2["activation_bytes_excl_adjacency"]),
            "fp32_excl_adjacency": mb(mem2["fp32_equivalent_excl_adjacency"]),
            "ratio_excl_adjacency": round(mem2["compression_ratio_excl_adjacency"], 3),
            "definition": "reference ledger (tape.py:86-93): quantized contexts + masks + indices + "
                          "margins; 'incl' also counts the shared CSR adjacency once (reference definition)"}
        out["epoch3_mean_loss"] = round(loss2, 5)
    if hbm_peak:
        out["hbm_step_peak_MB"] = {f"int{b}" if b != 32 else "fp32": round(v / 1e6, 3) for b, v in hbm_peak.items()}
        if 2 in hbm_peak and 32 in hbm_peak:
            out["hbm_step_peak_MB"]["ratio_fp32_over_int2"] = round(hbm_peak[32] / hbm_peak[2], 3)
        out["hbm_step_peak_MB"]["definition"] = (
            "torch.cuda.max_memory_allocated during one eager step (forward + backward, no Adam) "
            "minus the allocation before it: contexts, layer outputs, gradients and scratch; "
            "fp32 = the same engine at bits=32 (pass-through contexts)")
    return out


def quality_bench(args, shape=None):
    """Recall@20 / NDCG@20 after ``--quality-epochs`` full epochs from the
    reference's initial state (same params, batches, negatives: train_run,
    train.py:175-227) at INT2 (fast and compat noise) and FP32, next to the
    reference's own runs on the same dataset (datasets/*_reference_runs.json,
    written by datasets/run_reference_training.py in the build container)."""
    from paper_2212_04540_b200 import data as D
    import paper_2212_04540_b200 as kgq
    import torch
    from paper_2212_04540_b200.model import ModelConfig, embed
    from paper_2212_04540_b200.train import TrainConfig, evaluate, train_run
    shape = shape or args.train_shape
    ds = D.reference_dataset(shape)
    adj = D.build_adjacency(ds)
    out = {"epochs": args.quality_epochs, "dataset": f"{shape}_seed0 (reference generator)"}
    for name, bits, rng in (("int2_fast", 2, "fast"), ("int2_compat", 2, "compat"), ("fp32", 32, "fast")):
        q = kgq.QuantConfig(bits=bits, rng=rng)
        mcfg = ModelConfig(layers=3, dim=64, quant=q)
        params, rep = train_run(ds, mcfg, TrainConfig(epochs=args.quality_epochs, quant=q), adjacency=adj,
                                graphs=True)
        m = rep["metrics"]
        # train_run's eval_seconds is one call (whichever run comes first pays the
        # process's one-time setup); the steady-state cost: 3 more calls, median
        readout = embed(params, adj, mcfg)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.monotonic()
            evaluate(ds, readout, 20)
            torch.cuda.synchronize()
            ts.append(time.monotonic() - t0)
        out[name] = {"recall_at_20": round(m["recall_at_20"], 5), "ndcg_at_20": round(m["ndcg_at_20"], 5),
                     "loss_curve": [round(v, 6) for v in rep["loss_curve"]],
                     "epoch_s": [round(v, 3) for v in rep["timing"]["epoch_seconds"]],
                     "eval_s": round(rep["timing"]["eval_seconds"], 4),
                     "eval_s_steady": round(float(np.median(ts)), 4),
                     "activation_bytes_peak": rep["memory"]["activation_bytes_peak"]}
    ref_path = os.path.join(ROOT, "datasets", f"{shape}_seed0_reference_runs.json")
    if os.path.exists(ref_path):
        with open(ref_path) as f:
            ref = json.load(f)
        out["reference"] = {k: v for k, v in ref.items() if int(v.get("epochs", -1)) == args.quality_epochs}
    return out


def industry_bench(args):
    """BASELINE configs[4] (industry-scale KG, ~55M nodes, ~1e9 triples,
    d=128, 3 layers, INT2) as a ``world``-way row partition measured one rank
    at a time on this GPU: each simulated rank builds its own CSR row block
    from the device generator (industry.py), then runs the real per-rank
    partitioned step (parallel.partitioned_step, padded gather layout) with
    the collectives replaced by SimulatedRankComm (remote rows = stand-in
    values).  Reported: per-rank compute ms/step (max over the simulated
    ranks is the compute part of a W-GPU step), the exchange bytes per rank
    per step and their time at the measured NVLink peer bandwidth (an
    estimate, not a measurement), local activation ledger."""
    import torch
    import paper_2212_04540_b200 as kgq
    from paper_2212_04540_b200.industry import INDUSTRY, IndustryGraph
    from paper_2212_04540_b200.parallel import HaloPlan, RowPartition, SimulatedRankComm, partitioned_step
    from paper_2212_04540_b200.tensorops import CSR
    from paper_2212_04540_b200.train import AdamState, adam_step

    W = args.industry_world
    ranks = [int(r) for r in args.industry_ranks.split(",")]
    d, L, B = 128, 3, 1024
    t0 = time.perf_counter()
    g = IndustryGraph(INDUSTRY, seed=0, device="cuda")
    deg = g.degrees()
    cuts = g.partition(deg, W)
    torch.cuda.synchronize()
    t_deg = time.perf_counter() - t0
    U, I = INDUSTRY.users, INDUSTRY.items
    nnz_total = int(deg.sum())
    n_train = int(deg[:U].sum()) - U
    n_triples_edges = (nnz_total - g.n - 2 * n_train) // 2
    out = {"workload": f"industry-scale synthetic KG (device generator): {g.n} nodes ({U} users, {I} items, "
                       f"{INDUSTRY.entities} entities), {n_triples_edges} KG edges + {n_train} train pairs, "
                       f"adjacency nnz {nnz_total}; KGNN {L} layers d={d}, batch {B}, INT2 stochastic (fast rng)",
           "world": W, "generator_degrees_s": round(t_deg, 2), "ranks": {}}
    cfg = kgq.QuantConfig(bits=2, rng="fast")
    for rank in ranks:
        t1 = time.perf_counter()
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        ip, ix, vv = g.row_block(lo, hi, deg)
        part = RowPartition(W, rank, cuts, g.n)
        # halo ("boundary") exchange: receive only the remote rows this block
        # references, send the local rows the other ranks reference
        u = torch.unique(ix.long())
        remote = u[(u < lo) | (u >= hi)]
        del u
        owner = torch.searchsorted(torch.from_numpy(np.asarray(cuts, dtype=np.int64)).cuda(), remote,
                                   right=True) - 1
        recv_counts = torch.bincount(owner, minlength=W).cpu().tolist()
        send_counts = g.referenced_by_others(lo, hi, cuts).cpu().tolist()
        send_idx = torch.arange(int(sum(send_counts)), device="cuda", dtype=torch.int64) % (hi - lo)
        plan = HaloPlan(part, remote, recv_counts, send_counts, send_idx)   # volumes only (see below)
        # the step runs the all-gather-v layout: on this graph the halo is no
        # cheaper (item ranks reference ~all rows; attribute ranks receive 2M
        # rows but must pack and send 63M), so only its volumes are reported
        a_local = CSR(ip, ix, vv, (hi - lo, g.n), symmetric=False)      # global column ids
        del remote, owner, send_idx
        torch.cuda.synchronize()
        t_blk = time.perf_counter() - t1
        gen = torch.Generator(device="cuda").manual_seed(rank)
        bound = (6.0 / (g.n + d)) ** 0.5
        params = {"E0": (torch.rand((hi - lo, d), device="cuda", generator=gen) * 2 - 1) * bound}
        tb = (6.0 / (2 * d)) ** 0.5
        for i in range(L):
            params[f"theta{i}"] = (torch.rand((d, d), device="cuda", generator=gen) * 2 - 1) * tb
        state = AdamState(params)
        comm = SimulatedRankComm(W, rank)
        stream = kgq.RandomStream(0)
        users = torch.randint(0, U, (64, B), device="cuda", generator=gen)
        items = U + torch.randint(0, I, (64, 2, B), device="cuda", generator=gen)

        def one(k):
            th = [params[f"theta{i}"] for i in range(L)]
            loss, de0, dth = partitioned_step(part, a_local, params["E0"], th, users[k % 64],
                                              items[k % 64, 0], items[k % 64, 1], 1e-5, cfg, stream,
                                              comm, layout="global")
            grads = {"E0": de0}
            grads.update({f"theta{i}": t for i, t in enumerate(dth)})
            adam_step(params, grads, state, 1e-3)

        for k in range(max(args.warmup, 1)):
            one(k)
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_steps = max(1, min(args.steps, 5))
        a.record(cur)
        for k in range(n_steps):
            one(100 + k)
        b.record(cur)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n_steps
        if os.environ.get("KGQ_PROFILE_STEP"):     # ncu --profile-from-start off: one step
            torch.cuda.cudart().cudaProfilerStart()
            one(200)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
        rows = hi - lo
        out["ranks"][str(rank)] = {
            "rows": rows, "nnz": int(a_local.nnz), "block_build_s": round(t_blk, 2),
            "halo_rows": plan.n_halo, "halo_send_rows": int(sum(send_counts)),
            "halo_exchange_GB_per_step": round(2 * L * max(plan.recv_bytes(d), plan.send_bytes(d)) / 1e9, 2),
            "allgather_recv_GB_per_step": round(2 * L * (g.n - (hi - lo)) * d * 4 / 1e9, 2),
            "ms_per_step": round(ms, 2),
            "spmm_gathered_GB_per_step": round(2 * L * a_local.nnz * d * 4 / 1e9, 2),
            "activation_MB_local": round(L * rows * (d * 2 // 8 + 8 + d // 8) / 1e6, 1),
            "fp32_equivalent_MB_local": round(L * rows * (d * 4 + d // 8) / 1e6, 1),
            "peak_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1)}
        del a_local, ip, ix, vv, params, state, comm
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
    worst = max(v["ms_per_step"] for v in out["ranks"].values())
    # all-gather-v (layout="global"): every rank receives the rows it lacks,
    # 2L times per step; the largest receiver is the rank with fewest rows.
    # The halo alternative's volumes (max of send / receive) are beside it.
    xbytes = 2 * L * (g.n - min(int(cuts[r + 1] - cuts[r]) for r in range(W))) * d * 4
    halo = max(v["halo_exchange_GB_per_step"] for v in out["ranks"].values())
    out.update({"compute_ms_per_step_max_over_simulated_ranks": worst,
                "exchange": "all-gather-v of E and dH (layout='global'); max over the simulated ranks",
                "exchange_GB_per_rank_per_step": round(xbytes / 1e9, 2),
                "halo_exchange_GB_per_rank_per_step_max": halo,
                "steps_per_epoch": -(-n_train // B),
                "compute_hours_per_epoch_max_rank": round(-(-n_train // B) * worst / 3.6e6, 2),
                "note": "1-GPU box: per-rank compute measured one rank at a time (SIMULATED partition: "
                        "the other ranks' rows are stand-in values); collectives not timed and no peer "
                        "bandwidth measured here, so no exchange time or epoch time is claimed -- the "
                        "exchange is reported in bytes; with overlap=True the SpMM of source block p "
                        "runs while blocks p+1.. are in flight"})
    return out


def _partitioned_train_ms(ds, mcfg, cfg, stream, rng, world, rank, args):
    """Row-partitioned step timing (parallel.partitioned_step over NCCL)."""
    import torch
    from paper_2212_04540_b200 import data as D
    from paper_2212_04540_b200.model import init_params
    from paper_2212_04540_b200.parallel import Comm, GpuOps, RowPartition, partitioned_step
    indptr, indices, vals = D.adjacency_arrays(ds)
    part = RowPartition.build(indptr, world, rank)
    layout = part.preferred_layout()
    a_local = GpuOps.local_adjacency(indptr, indices, vals, part.lo, part.hi, ds.num_nodes, "cuda",
                                     part=part if layout == "padded" else None)
    # all-gather-v layout: the SpMM runs source block by source block as the
    # broadcasts land (parallel.partitioned_step overlap=True), plan built once
    overlap = layout == "global" and not args.no_overlap
    plan = GpuOps.overlap_plan(a_local, part.cuts) if overlap else None
    from paper_2212_04540_b200.train import AdamState, adam_step
    params = init_params(ds.num_nodes, mcfg, 0)
    local = {"E0": params.entity_embeddings[part.lo:part.hi].clone()}
    for i, t in enumerate(params.layer_weights):
        local[f"theta{i}"] = t
    state = AdamState(local)
    comm = Comm()
    trip = torch.from_numpy(D.sample_negatives(ds, rng)).cuda().long()
    n_users = ds.num_users
    n_full = len(trip) // 1024

    def one(i):
        b = trip[(i % n_full) * 1024:][:1024]
        thetas = [local[f"theta{k}"] for k in range(mcfg.layers)]
        loss, de0, dth = partitioned_step(part, a_local, local["E0"], thetas, b[:, 0], n_users + b[:, 1],
                                          n_users + b[:, 2], cfg.l2, cfg.quant, stream, comm, layout=layout,
                                          overlap=overlap, plan=plan)
        grads = {"E0": de0}
        grads.update({f"theta{k}": g for k, g in enumerate(dth)})
        adam_step(local, grads, state, cfg.lr)

    for i in range(args.warmup + 2):
        one(i)
    torch.cuda.synchronize()
    sg = None
    if not args.no_graphs:      # the step with its collectives captured once (eager fallback)
        from paper_2212_04540_b200.parallel import PartitionedStepGraph
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                sg = PartitionedStepGraph(part, a_local, local, state, cfg, stream, comm, mcfg.layers, 1024,
                                          args.train_steps + 2, layout=layout, overlap=overlap, plan=plan)
            torch.cuda.current_stream().wait_stream(side)
        except Exception as exc:      # noqa: BLE001 - keep the eager number
            print(f"[bench] partitioned graph capture failed ({type(exc).__name__}: {exc}); eager", file=sys.stderr)
            sg = None
    batches = [(trip[(i % n_full) * 1024:][:1024, 0], n_users + trip[(i % n_full) * 1024:][:1024, 1],
                n_users + trip[(i % n_full) * 1024:][:1024, 2]) for i in range(100, 100 + args.train_steps)]
    if sg is not None:
        sg.run(batches[:2], stream, state)
    torch.cuda.synchronize()
    barrier(world)
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    if sg is not None:
        sg.run(batches, stream, state)
    else:
        for i in range(args.train_steps):
            one(100 + i)
    b.record(cur)
    torch.cuda.synchronize()
    return max_over_ranks(a.elapsed_time(b) / args.train_steps, world)


def run_ours(args):
    import torch
    world, rank, local = dist_setup(args)
    import paper_2212_04540_b200 as kgq
    from paper_2212_04540_b200 import _lib

    rows, cols, bits, group = args.rows, args.cols, args.bits, args.group
    free, _ = torch.cuda.mem_get_info()
    need = rows * cols * 4 * 2.3
    if need > free:
        rows = int(rows * free / need) // 1024 * 1024
    n = rows * cols
    bpe = algo_bytes_per_elem(bits, group)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn((rows, cols), device="cuda", generator=g)
    cfg = kgq.QuantConfig(bits=bits, group=group, rng=args.rng)
    stream = kgq.RandomStream(1)
    row_off = rank * rows
    goff = row_off * cols // group

    def step(tid):
        q = kgq.quantize_tensor(x, cfg, stream, tensor_id=tid, group_offset=goff)
        out = kgq.dequantize_tensor(q)
        return q, out

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(cur)
        for s in range(args.steps):
            e0, e1, e2 = ev[s]
            e0.record(cur)
            q = kgq.quantize_tensor(x, cfg, stream, tensor_id=100 + s, group_offset=goff)
            e1.record(cur)
            out = kgq.dequantize_tensor(q)
            e2.record(cur)
            del q, out
        t_end.record(cur)
        torch.cuda.synchronize()
    barrier(world)
    ms_total = t_start.elapsed_time(t_end)
    ms_total = max_over_ranks(ms_total, world)
    q_ms = [e0.elapsed_time(e1) for e0, e1, _ in ev]
    d_ms = [e1.elapsed_time(e2) for _, e1, e2 in ev]
    peak, peak_src = load_peaks()
    step_bytes = 2 * n * bpe
    value = world * step_bytes * args.steps / (ms_total / 1e3) / 1e9
    q_avg = sum(q_ms) / len(q_ms)
    d_avg = sum(d_ms) / len(d_ms)
    q_gbs = n * bpe / (q_avg / 1e3) / 1e9
    d_gbs = n * bpe / (d_avg / 1e3) / 1e9
    traffic = load_traffic()

    # compat-stream (reference-identical noise) quantize, a few launches
    comp = None
    if not args.skip_compat:
        ccfg = kgq.QuantConfig(bits=bits, group=group, rng="compat")
        kgq.quantize_tensor(x, ccfg, stream, tensor_id=7)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for s in range(3):
            kgq.quantize_tensor(x, ccfg, stream, tensor_id=200 + s, group_offset=goff)
        b.record(cur)
        torch.cuda.synchronize()
        c_ms = a.elapsed_time(b) / 3
        comp = {"quantize_ms": round(c_ms, 3), "quantize_GBps": round(n * bpe / (c_ms / 1e3) / 1e9, 1),
                "frac": round(n * bpe / (c_ms / 1e3) / 1e9 / peak, 4)}

    # end to end through the public API with host buffers (pinned), a
    # bounded slice of the workload: H2D of the fp32 activations, quantize,
    # dequantize, D2H of the reconstructed activations, every step.
    e2e = None
    if not args.skip_e2e:
        e_rows = min(rows, args.e2e_rows)
        xh = torch.empty((e_rows, cols), dtype=torch.float32, pin_memory=True)
        xh.copy_(x[:e_rows].cpu())
        oh = torch.empty_like(xh, pin_memory=True)
        del x
        torch.cuda.empty_cache()

        # the step is pipelined over row chunks on 3 streams, so the H2D of
        # chunk c+1 overlaps the kernels of chunk c and the D2H of chunk c-1
        # (PCIe is full duplex); the noise is keyed by global group index,
        # so the chunked result is byte-identical to one call.
        side = [torch.cuda.Stream() for _ in range(3)]
        n_ch = max(1, min(args.e2e_chunks, e_rows // 1024))
        step_rows = -(-e_rows // n_ch // 1024) * 1024
        bounds = [(r0, min(e_rows, r0 + step_rows)) for r0 in range(0, e_rows, step_rows)]

        def e2e_step(tid):
            go = torch.cuda.Event()
            go.record(cur)
            for c, (r0, r1) in enumerate(bounds):
                sc = side[c % len(side)]
                sc.wait_event(go)
                with torch.cuda.stream(sc):
                    xd = xh[r0:r1].to("cuda", non_blocking=True)
                    q = kgq.quantize_tensor(xd, cfg, stream, tensor_id=tid,
                                            group_offset=goff + r0 * cols // group)
                    out = kgq.dequantize_tensor(q)
                    oh[r0:r1].copy_(out, non_blocking=True)
            for sc in side:
                cur.wait_stream(sc)

        for w in range(2):
            e2e_step(300 + w)
        torch.cuda.synchronize()
        if len(bounds) > 1:   # chunk seam == one unchunked call (byte-identical)
            r0 = bounds[1][0] - 512
            xs = xh[r0:r0 + 1024].to("cuda")
            ref = kgq.dequantize_tensor(kgq.quantize_tensor(xs, cfg, stream, tensor_id=301,
                                                            group_offset=goff + r0 * cols // group))
            if not torch.equal(ref.cpu(), oh[r0:r0 + 1024]):
                raise RuntimeError("pipelined e2e result differs from the unchunked call")
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        ke = max(2, min(args.steps, 5))
        for s in range(ke):
            e2e_step(400 + s)
        b.record(cur)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(a.elapsed_time(b), world)
        e_val = world * 2 * e_rows * cols * bpe * ke / (e_ms / 1e3) / 1e9
        # the reference's calling convention: host tensor in, host context
        # out, then host context in, host tensor out (kgq_*_host_f32; each
        # call pipelines its own chunks and blocks like the numpy call)
        import time as _time
        ctx = kgq.empty_context(e_rows, cols, cfg, pin_memory=True)
        qh = kgq.quantize_tensor(xh, cfg, stream, tensor_id=500, out=ctx)
        oh2 = kgq.dequantize_tensor(qh, out=oh)
        t0 = _time.perf_counter()
        for s in range(ke):
            qh = kgq.quantize_tensor(xh, cfg, stream, tensor_id=510 + s, group_offset=goff, out=ctx)
            oh2 = kgq.dequantize_tensor(qh, out=oh)
        h_s = _time.perf_counter() - t0
        host_api = {"value": round(2 * e_rows * cols * bpe * ke / h_s / 1e9, 3), "unit": UNIT,
                    "calls": "quantize_tensor(host, out=pinned ctx) -> dequantize_tensor(host ctx, "
                             "out=pinned), blocking, wall clock"}
        del qh, oh2, ctx
        link = pcie_probe(xh, oh)
        # the e2e step moves 4 B/elem each way at once: its link-bound ceiling
        # is the slower direction of the simultaneous two-stream copy
        ceil_s = max(e_rows * cols * 4 / (link["both_h2d_GBps"] * 1e9),
                     e_rows * cols * 4 / (link["both_d2h_GBps"] * 1e9))
        link["e2e_ceiling"] = round(2 * e_rows * cols * bpe / ceil_s / 1e9, 3)
        link["e2e_frac_of_link"] = round(e_val / world / link["e2e_ceiling"], 4)
        e2e = {"value": round(e_val, 3), "unit": UNIT, "h2d_bytes_per_step": e_rows * cols * 4,
               "d2h_bytes_per_step": e_rows * cols * 4,
               "sample": f"{e_rows}x{cols} fp32 per GPU per step (pinned host buffers), "
                         f"{len(bounds)} row chunks pipelined on 3 streams through "
                         f"quantize_tensor/dequantize_tensor",
               "host_api": host_api, "link": link}

    train = None
    if not args.skip_train:
        torch.cuda.empty_cache()
        try:
            train = train_bench(args, world, rank)
        except Exception as exc:            # never lose the headline line
            train = {"error": f"{type(exc).__name__}: {exc}"}
        if world == 1 and args.train_shape == "amazon" and not args.skip_lastfm:
            torch.cuda.empty_cache()
            try:      # BASELINE configs[2]: the Last-FM-shaped KG on one B200
                train["lastfm"] = train_bench(args, world, rank, shape="lastfm", with_fp32=False,
                                              with_cpu=False)
            except Exception as exc:
                train["lastfm"] = {"error": f"{type(exc).__name__}: {exc}"}
        if world == 1 and not args.skip_quality and args.train_shape in ("amazon", "lastfm"):
            torch.cuda.empty_cache()
            try:
                train["quality"] = quality_bench(args)
            except Exception as exc:
                train["quality"] = {"error": f"{type(exc).__name__}: {exc}"}
            if args.train_shape == "amazon" and isinstance(train.get("lastfm"), dict) and \
                    os.path.exists(os.path.join(ROOT, "datasets", "lastfm_seed0_reference_runs.json")):
                torch.cuda.empty_cache()
                try:      # configs[2] quality next to the reference's own Last-FM runs
                    train["lastfm"]["quality"] = quality_bench(args, shape="lastfm")
                except Exception as exc:
                    train["lastfm"]["quality"] = {"error": f"{type(exc).__name__}: {exc}"}

    verification = None
    if world == 1 and not args.skip_verification:
        # SURVEY 8(a) a18 at the reference's full scale (quantize.py:358-412:
        # 100 rows x d=64 x 1e5 draws x 4 widths), every draw through K1
        torch.cuda.empty_cache()
        try:
            from paper_2212_04540_b200 import verification as V
            verification = {"scale": "100 rows x d=64 x 1e5 draws x bits 1/2/4/8, seed 0 (the reference's sweep)",
                            "reference_seconds": 25.3,
                            "reference_source": "pkg/test_output.txt:10 (SURVEY.md 8(a) a18)",
                            "note": "criterion (a) is a fixed-seed 4-sigma test over 6,400 elements per width; "
                                    "over seeds 0-11 it trips in 3/48 (fast) and 5/48 (compat = numpy's "
                                    "Philox4x64-10) cells (profiles/r1_verification_seeds.json)"}
            for rng_name in ("fast", "compat"):
                t0 = time.perf_counter()
                rep = V.quantizer_verification(bits_list=(1, 2, 4, 8), n_rows=100, dim=64, trials=100000,
                                               seed=0, rng=rng_name)
                torch.cuda.synchronize()
                verification[rng_name] = {
                    "passed": rep["passed"], "seconds": round(time.perf_counter() - t0, 2),
                    "bits": {str(b): {k: round(v, 4) if isinstance(v, float) else v for k, v in e.items()}
                             for b, e in rep["bits"].items()}}
        except Exception as exc:
            verification = {"error": f"{type(exc).__name__}: {exc}"}

    industry = None
    if args.industry and world == 1:
        torch.cuda.empty_cache()
        try:
            industry = industry_bench(args)
        except Exception as exc:
            industry = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        threads = os.cpu_count() or 1
        gbs, el, reps = cpu_port_run(args.cpu_rows, cols, bits, group, threads, min_seconds=10.0,
                                     max_reps=50, rng=args.rng)
        c_gbs, c_el, c_reps = cpu_port_run(args.cpu_rows, cols, bits, group, threads, min_seconds=5.0,
                                           max_reps=20, rng="compat")
        cpu = {"value": round(gbs, 4), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{reps} x ({args.cpu_rows}x{cols} fp32 quantize+dequantize, rng={args.rng} as "
                         f"in config) in {el:.1f}s; oracle/kgq_oracle.c, pthreads",
               "value_rng_compat": round(c_gbs, 4),
               "sample_rng_compat": f"{c_reps} x ({args.cpu_rows}x{cols}), the reference's numpy "
                                    f"Philox4x64-10 stream, in {c_el:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_total / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch.randn fp32 activations)",
            "config": dict(workload_config(args), rows_per_gpu=rows,
                           parallelism=f"row shards x{world}, no data-path collective"),
            "frac_of_peak": round(value / world / peak, 4),
            "roofline": {"bound": "hbm", "kernel": "quantize_fast_kernel (K1, fused quantize+pack)",
                         "achieved": round(q_gbs, 1), "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": round(q_gbs / peak, 4),
                         "traffic": (round(traffic["quantize"]["dram_bytes_per_elem"] * n)
                                     if "quantize" in traffic else None),
                         "traffic_note": "dram__bytes_read+write per element from the committed ncu "
                                         "capture (profiles/traffic.json), scaled to this launch",
                         "algorithmic_bytes_per_launch": int(n * bpe)},
            "kernels": {
                "quantize": {"ms": round(q_avg, 4), "GBps": round(q_gbs, 1), "frac": round(q_gbs / peak, 4)},
                "dequantize": {"ms": round(d_avg, 4), "GBps": round(d_gbs, 1), "frac": round(d_gbs / peak, 4),
                               "traffic": (round(traffic["dequantize"]["dram_bytes_per_elem"] * n)
                                           if "dequantize" in traffic else None)},
                "quantize_compat_rng": comp,
            },
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "train": train,
            **({"industry": industry} if industry is not None else {}),
            **({"verification": verification} if verification is not None else {}),
            "native_lib": os.path.relpath(_lib.LIB_PATH, ROOT),
        }
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    return 0


def launch(args, argv):
    """``bench.py --gpus N`` starts its own N ranks, one process per GPU:
    under torchrun (WORLD_SIZE set) this process is one rank and runs; with
    N > 1 and no torchrun it re-executes itself through
    ``torch.distributed.run`` (127.0.0.1 rendezvous, the driver's own launch
    line) and returns the launcher's exit code -- rank 0 prints the one JSON
    line; N == 1 runs in this process (world 1, the same code path).
    Returns None when this process should run the benchmark itself."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return None
    import socket
    with socket.socket() as sk:                   # a free rendezvous port
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    if not args.launch_selftest:                  # NCCL communicator setup (NVLS / ring / tree) in the log
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import subprocess
    return subprocess.call(cmd, env=env)


def launch_selftest(args):
    """The launcher's plumbing without a GPU (gloo): every rank times a
    rank-dependent sleep between barriers, the max over ranks goes to rank 0,
    which prints the line a real run would (n_gpus = world)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "selftest": True, "n_gpus": world, "steps": args.steps,
                          "max_rank_seconds": round(float(t.item()), 4),
                          "ranks_seen": world}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rows", type=int, default=64 << 20)
    ap.add_argument("--cols", type=int, default=128)
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--group", type=int, default=64)
    ap.add_argument("--rng", default="fast", choices=["fast", "compat"])
    ap.add_argument("--e2e-rows", type=int, default=8 << 20)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--cpu-rows", type=int, default=1 << 20)
    ap.add_argument("--ref-rows", type=int, default=2 << 20)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-compat", action="store_true")
    ap.add_argument("--skip-train", action="store_true")
    ap.add_argument("--skip-quality", action="store_true")
    ap.add_argument("--skip-lastfm", action="store_true")
    ap.add_argument("--skip-verification", action="store_true")
    ap.add_argument("--industry", action="store_true", help="configs[4] per-rank shard measurement")
    ap.add_argument("--industry-world", type=int, default=8)
    ap.add_argument("--industry-ranks", default="0")
    ap.add_argument("--quality-epochs", type=int, default=1)
    ap.add_argument("--no-graphs", action="store_true", help="train step without CUDA graphs")
    ap.add_argument("--no-overlap", action="store_true", help="partitioned step: exchange, then compute")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the row-partitioned (multi-GPU) training step even at 1 GPU")
    ap.add_argument("--train-shape", default="amazon", choices=["small", "lastfm", "amazon"])
    ap.add_argument("--train-steps", type=int, default=100)
    ap.add_argument("--launch-selftest", action="store_true",
                    help="exercise the --gpus N launcher on CPU (gloo), no benchmark")
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    rc = launch(args, argv)
    if rc is not None:
        return rc
    if args.launch_selftest:
        return launch_selftest(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.warmup < 3 and args.impl == "ours" and not os.environ.get("KGQ_ALLOW_SHORT_WARMUP"):
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
