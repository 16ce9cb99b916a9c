#!/bin/bash
# A/B of variant-path builds (abl/H.so baseline, abl/G32.so, abl/G16.so): variant GPU tests, then (iii)(b)/(c) run times on 50M mixed hits.
LIB=paper_2412_11809_b200/lib/libtpxcluster.so
cp abl/G16.so $LIB
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/var_pt.log 2>&1; echo "pytest(G16)=$?"; tail -1 gpurun_out/var_pt.log
cp abl/G32.so $LIB
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -k "not slow" > gpurun_out/var_pt32.log 2>&1; echo "pytest(G32)=$?"; tail -1 gpurun_out/var_pt32.log
for r in 1 2; do for v in H G32 G16; do
cp abl/$v.so $LIB
python - <<PY
import sys, time, numpy as np, torch
sys.path.insert(0,'.')
import tpxgen, paper_2412_11809_b200 as tpx
h = tpxgen.generate('mixed', n_hits=50_000_000)
d = torch.from_numpy(h.view(np.uint8)).cuda()
for vname, vv in (('global', tpx.VARIANT_GLOBAL), ('static', tpx.VARIANT_STATIC)):
    c = tpx.Clusterer(320, variant=vv)
    for _ in range(2): c.run(d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): _, _, k = c.run(d)
    e1.record(); torch.cuda.synchronize()
    print('$v$r', vname, round(e0.elapsed_time(e1)/3, 3), 'ms', k)
PY
done; done
cp abl/G16.so $LIB
