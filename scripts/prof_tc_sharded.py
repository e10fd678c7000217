"""Triangle count through the sharded orientation (distributed.orient +
gt_triangles_oriented_part) at world size 1 on a BASELINE config, with the
library's per-phase device times, next to the single-GPU path."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1503_07881_b200 as gt  # noqa: E402
from paper_1503_07881_b200 import _native  # noqa: E402
from paper_1503_07881_b200 import distributed as D  # noqa: E402
from paper_1503_07881_b200.synth import CONFIGS, rmat_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
os.environ["MASTER_ADDR"] = "127.0.0.1"
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
ops = D.NativeOps("cuda:0")
src, dst = rmat_device(CONFIGS[cfg])
sg = D.build_csr(src, dst, ops=ops)
del src, dst


def phases(tag, fn):
    _native.profile_reset()
    _native.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ph = _native.profile_read()
    _native.profile_enable(False)
    print(f"{tag}: {dt*1e3:.1f} ms", flush=True)
    for k, (ms, cnt, by) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:24s} {ms:8.2f} ms  x{cnt}", flush=True)
    return r


for i in range(reps):
    off_p, adj_p = phases(f"rep {i} orient (sharded)", lambda: D.orient(sg, ops=ops))
    c = phases(f"rep {i} count", lambda: ops.triangles_oriented_part(off_p, adj_p, 0, 1))
    print(f"rep {i}: triangles {c}", flush=True)
    del off_p, adj_p
dist.destroy_process_group()
