"""Host<->device copy ceilings for the e2e leg (pinned, 4 GiB): H2D alone,
D2H alone, and both directions at once on two streams."""
import json
import torch

n = 1 << 30                                   # floats (4 GiB)
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    for s, f in ((s1, lambda: d_in.copy_(h_in, non_blocking=True)),
                 (s2, lambda: h_out.copy_(d_out, non_blocking=True))):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            f()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


gb = n * 4 / 1e9
h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
bi = timed(both)
print(json.dumps({"h2d_GBps": round(gb / h2d * 1e3, 1), "d2h_GBps": round(gb / d2h * 1e3, 1),
                  "bidirectional_each_GBps": round(gb / bi * 1e3, 1), "bytes_each": n * 4}))
