"""BASELINE configs[1] sweep (not the headline bench line): quantize and
dequantize throughput for fp32 rows in {1M, 4M, 16M, 64M} x cols {64, 128},
INT2/INT4/INT8, group 64/256, fast noise (plus quantize with the reference's
Philox4x64-10 stream, rng="compat"); algorithmic bytes / CUDA-event time vs
the measured HBM peak.  Output: one JSON document."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_04540_b200 as kgq

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
res = []
for rows in (1 << 20, 4 << 20, 16 << 20, 64 << 20):
    for cols in (64, 128):
        if rows * cols > (64 << 20) * 128:
            continue
        x = torch.randn(rows, cols, device="cuda")
        for bits in (2, 4, 8):
            for group in (64, 256):
                cfg = kgq.QuantConfig(bits=bits, group=group, rng="fast")
                st = kgq.RandomStream(1)
                q = kgq.quantize_tensor(x, cfg, st, tensor_id=0)
                out = kgq.dequantize_tensor(q)
                torch.cuda.synchronize()
                n = rows * cols
                bpe = 4 + bits / 8 + 8 / group
                reps = max(3, int(2e9 / (n * bpe)))
                for r in range(reps):          # warm the allocator at this size (untimed)
                    q = kgq.quantize_tensor(x, cfg, st, tensor_id=1 + r)
                    out = kgq.dequantize_tensor(q)
                torch.cuda.synchronize()
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record()
                for r in range(reps):
                    q = kgq.quantize_tensor(x, cfg, st, tensor_id=1 + r)
                b.record()
                for r in range(reps):
                    out = kgq.dequantize_tensor(q)
                c.record()
                torch.cuda.synchronize()
                tq, td = a.elapsed_time(b) / reps, b.elapsed_time(c) / reps
                gq, gd = n * bpe / tq / 1e6, n * bpe / td / 1e6
                ccfg = kgq.QuantConfig(bits=bits, group=group, rng="compat")
                creps = max(2, reps // 4)
                q = kgq.quantize_tensor(x, ccfg, st, tensor_id=0)
                torch.cuda.synchronize()
                a.record()
                for r in range(creps):
                    q = kgq.quantize_tensor(x, ccfg, st, tensor_id=1 + r)
                b.record()
                torch.cuda.synchronize()
                gc = n * bpe / (a.elapsed_time(b) / creps) / 1e6
                res.append({"rows": rows, "cols": cols, "bits": bits, "group": group,
                            "quantize_GBps": round(gq, 1), "quantize_frac": round(gq / peak, 4),
                            "dequantize_GBps": round(gd, 1), "dequantize_frac": round(gd / peak, 4),
                            "quantize_compat_GBps": round(gc, 1), "quantize_compat_frac": round(gc / peak, 4)})
                print(res[-1], flush=True)
                del q, out
        del x
        torch.cuda.empty_cache()
print(json.dumps({"peak_GBps": peak, "rng": "fast (quantize_compat_*: rng=compat)", "sweep": res}))
