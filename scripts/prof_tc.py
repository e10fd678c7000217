"""Triangle count on a BASELINE config's graph, `reps` times: per-phase
device times (the command ncu captures for the count kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_07881_b200 as gt  # noqa: E402
from paper_1503_07881_b200 import _native  # noqa: E402
from paper_1503_07881_b200.synth import CONFIGS, rmat_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
src, dst = rmat_device(CONFIGS[cfg])
g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
del src, dst
for i in range(reps):
    _native.profile_reset()
    _native.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tc = gt.triangle_count(g)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ph = _native.profile_read()
    _native.profile_enable(False)
    print(f"rep {i}: triangles {tc} in {dt*1e3:.1f} ms", flush=True)
    for k, (ms, cnt, by) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:24s} {ms:8.2f} ms  x{cnt}", flush=True)
