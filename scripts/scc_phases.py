"""Per-phase device time of one call of each CSR consumer on a config's graph (diagnostic)."""
import sys

import torch

import paper_1503_07881_b200 as gt
from paper_1503_07881_b200 import _native
from paper_1503_07881_b200.synth import CONFIGS, rmat_device

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
src, dst = rmat_device(spec)
g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
del src, dst
gt.scc(g)
src0 = int(g.csr().ids[0])
for name, fn in (("scc", gt.scc), ("sssp", lambda x: gt.sssp(x, src0)),
                 ("cc", gt.connected_components), ("kcore8", lambda x: gt.k_core(x, 8))):
    _native.profile_reset()
    _native.profile_enable(True)
    fn(g)
    torch.cuda.synchronize()
    ph = _native.profile_read()
    _native.profile_enable(False)
    for k, v in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"{name} {k:20s} {v[0]:9.3f} ms  {v[1]:6d} launches")
