"""Do two clustering runs on two streams (host threads) overlap on the GPU?
Compares 2 sequential runs with 2 concurrent runs (separate contexts,
workspaces and streams) on the mixed preset."""
import sys, threading, time
import numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
h = tpxgen.generate("mixed", n_hits=n)
dev = torch.device("cuda:0")
d = [torch.from_numpy(h.view(np.uint8)).to(dev) for _ in range(2)]
ctx = [tpx.Clusterer(320) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
outs = []
for i in range(2):
    for _ in range(2):
        ctx[i].run(d[i], stream=streams[i])
torch.cuda.synchronize()

def one(i):
    with torch.cuda.stream(streams[i]):
        ctx[i].run(d[i], stream=streams[i])

for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    one(0); one(1)
    torch.cuda.synchronize(); seq = time.perf_counter() - t
    t = time.perf_counter()
    th = [threading.Thread(target=one, args=(i,)) for i in range(2)]
    [x.start() for x in th]; [x.join() for x in th]
    torch.cuda.synchronize(); con = time.perf_counter() - t
    print(f"n={n}: sequential {seq*1e3:.2f} ms, concurrent {con*1e3:.2f} ms, ratio {con/seq:.3f}")
