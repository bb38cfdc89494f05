"""PCIe copy bound of the config-2 e2e step (development aid).

Times, with CUDA events, the step's copies alone from/to pinned host memory:
25 MB of query positions H2D, 9.4 MB of (w, status) D2H, and both at once on
two streams -- the floor of an end-to-end eval that moves those bytes.
"""
import json

import torch

n = 1 << 20
dev = torch.device("cuda:0")
h_in = torch.empty(3 * n, dtype=torch.float64).pin_memory()
h_w = torch.empty(n, dtype=torch.float64).pin_memory()
h_st = torch.empty(n, dtype=torch.int8).pin_memory()
d_in = torch.empty(3 * n, dtype=torch.float64, device=dev)
d_w = torch.empty(n, dtype=torch.float64, device=dev)
d_st = torch.empty(n, dtype=torch.int8, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_w.copy_(d_w, non_blocking=True)
    h_st.copy_(d_st, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    with torch.cuda.stream(s_in):
        h2d()
    with torch.cuda.stream(s_out):
        d2h()
    cur.wait_stream(s_in)
    cur.wait_stream(s_out)


t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
print(json.dumps({
    "h2d_ms": t_in, "h2d_GBps": 24 * n / t_in / 1e6,
    "d2h_ms": t_out, "d2h_GBps": 9 * n / t_out / 1e6,
    "both_ms": t_both,
    "e2e_bound_queries_per_s": n / (t_both * 1e-3),
}))
