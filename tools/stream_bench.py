"""Host-to-host throughput of tpx_stream_run_host on a mixed stream (pinned input)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
bufs = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["20000000", "50000000"])]
hh = torch.empty(n * 16, dtype=torch.uint8).pin_memory()
tpxgen.generate("mixed", n_hits=n, out=hh.numpy())
h = hh.numpy().view(tpxgen.HIT_DTYPE)
toa = h["toa"].astype(np.int64)
t_dis = int(max(0, (np.maximum.accumulate(toa)[:-1] - toa[1:]).max())) + 1
del toa
order = torch.empty(n, dtype=torch.int32).pin_memory()
cl = torch.empty((n // 4, 80), dtype=torch.uint8).pin_memory()
for b in bufs:
    r = tpx.StreamRunner(320, b, b // 20, t_dis, 64, max_device_hits=b + b // 10)
    r.run(hh, order, cl)  # warm-up
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        k = r.run(hh, order, cl)
        times.append(time.perf_counter() - t0)
    st = r.last_stats
    print(f"b={b}: host-to-host {n / min(times) / 1e6:.0f} Mhit/s (best of 3, {min(times)*1e3:.1f} ms), "
          f"device span {n / (st['device_ms'] * 1e-3) / 1e6:.0f} Mhit/s, k={k}, buffers={st['buffers']}, "
          f"carried_max={st['carried_max']}, late={st['late_hits']}")
    del r
    torch.cuda.empty_cache()
