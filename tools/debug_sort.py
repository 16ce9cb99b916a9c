"""Debug helper: inspect workspace intermediates after a run (layout mirror)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen, oracle
import paper_2412_11809_b200 as tpx

def a256(v): return (v + 255) & ~255

def layout(n):
    off = 0; L = {}
    for name, b in [("hdr", 64), ("keys0", n*8), ("keys1", n*8), ("vals0", n*4), ("vals1", n*4), ("rec", n*16), ("parent", n*4), ("minidx", n*4)]:
        L[name] = off; off += a256(b)
    return L

for n in [int(a) for a in sys.argv[1:]] or [4096, 4097, 8191]:
    h = tpxgen.generate("mixed", n_hits=n)
    c = tpx.Clusterer(320)
    d = torch.from_numpy(h.view(np.uint8)).cuda()
    ws = torch.zeros(c.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    labels, feats, k = c.run(d, workspace=ws)
    torch.cuda.synchronize()
    L = layout(n)
    w = ws.cpu().numpy()
    rec = w[L["rec"]:L["rec"]+n*16].view(np.uint64).reshape(n, 2)
    toa = rec[:, 0] >> np.uint64(16)
    idx = (rec[:, 1] >> np.uint64(32)).astype(np.int64)
    ref_perm = np.lexsort((np.arange(n), h["toa"].astype(np.int64)))
    rl, rf = oracle.cluster(h, 320)
    gl = labels.cpu().numpy().view(np.uint32)
    print(n, "k", k, "ref", len(rf), "sorted", bool(np.all(np.diff(toa.astype(np.int64)) >= 0)),
          "perm==ref", bool(np.array_equal(idx, ref_perm)), "labels bad", int((gl != rl).sum()),
          "rec toa == hit toa", bool(np.array_equal(toa, h["toa"][idx])))
    if not np.array_equal(idx, ref_perm):
        bad = np.nonzero(idx != ref_perm)[0]
        print("  first bad positions", bad[:10], idx[bad[:10]], ref_perm[bad[:10]])
