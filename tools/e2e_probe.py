"""Host-buffer path probe: the copy floor of one step's transfers (H2D of the
hits, D2H of labels + records, pipelined across steps on two copy streams)
vs tpx_pipeline at several depths / step counts.   python tools/e2e_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2412_11809_b200 as tpx
import tpxgen

n = 200_000_000
k_rec = 29_778_330
h_host = torch.empty(n * 16, dtype=torch.uint8).pin_memory()
tpxgen.generate("mixed", n_hits=n, out=h_host.numpy())

# ---- copy floor: step i = H2D(hits) on s_in, then D2H(labels + records) on s_out
d_in = [torch.empty(n * 16, dtype=torch.uint8, device="cuda") for _ in range(2)]
d_out = torch.empty(n * 4 + k_rec * 64, dtype=torch.uint8, device="cuda")
h_out = torch.empty(n * 4 + k_rec * 64, dtype=torch.uint8).pin_memory()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
for steps in (6, 12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s_in)
    s_out.wait_event(e0)
    for i in range(steps):
        with torch.cuda.stream(s_in):
            d_in[i % 2].copy_(h_host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        s_out.wait_event(ev)
        with torch.cuda.stream(s_out):
            h_out.copy_(d_out, non_blocking=True)
    e1.record(s_out)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"copy floor, {steps} steps: {ms:.1f} ms/step = {n / ms / 1e3:.0f} Mhit/s", flush=True)
del d_in, d_out, h_out
torch.cuda.empty_cache()

cap = n // 4
for depth in (2, 3, 4):
    lab = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(depth)]
    ft = [torch.empty((cap, 64), dtype=torch.uint8).pin_memory() for _ in range(depth)]
    for steps in (6, 12):
        ms, k = bench._e2e(tpx, 320, n, h_host, lab, ft, cap, depth, steps)
        print(f"pipeline depth {depth}, {steps} steps: {ms:.1f} ms/step = {n / ms / 1e3:.0f} Mhit/s (k={k})", flush=True)
    del lab, ft
