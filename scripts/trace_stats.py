"""Per-role event-pair time totals of CTA 0 for a trace build (ADASGD_LIB=..._trace.so); tools only."""
import collections
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen
from paper_2110_07029_b200.api import Replica

cfg = synthgen.CONFIGS["amazon670k"]
ds = synthgen.make_dataset(cfg, n=20000)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
              max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.01, precision="bf16")
rep.upload_dataset(ds)
lib = rep.lib
buf = np.zeros((16384, 3), np.int64)
for k in range(3):
    lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False); torch.cuda.synchronize()
n = lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
ev = buf[:n]
# roles are concatenated in order; split where the clock goes backwards
roles, cur = [], [ev[0]]
for e in ev[1:]:
    if e[0] < cur[-1][0]:
        roles.append(cur); cur = []
    cur.append(e)
roles.append(cur)
t0 = min(r[0][0] for r in roles)
print(os.path.basename(os.environ.get("ADASGD_LIB", "")), "events", n)
for ri, r in enumerate(roles):
    span = r[-1][0] - r[0][0]
    pairs = collections.defaultdict(lambda: [0, 0])
    for a, b in zip(r[:-1], r[1:]):
        k = (int(a[1]), int(b[1]))
        pairs[k][0] += 1; pairs[k][1] += int(b[0] - a[0])
    print("role %d: first %+d last %+d span %d cycles" % (ri, r[0][0] - t0, r[-1][0] - t0, span))
    for k, (c, t) in sorted(pairs.items(), key=lambda kv: -kv[1][1])[:8]:
        print("   %2d->%2d  n=%5d  total=%9d (%5.1f%%)  mean=%7.1f" % (k[0], k[1], c, t, 100.0 * t / max(span, 1), t / c))
