"""CTA 0's pass-2 event timeline on the trace build (ADASGD_LIB=..._trace.so) for one
config (argv[1]); tools only.  Prints every event relative to the first, per role."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen
from paper_2110_07029_b200.api import Replica

cfg = synthgen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "amazoncat13k"]
ds = synthgen.make_dataset(cfg, n=20000)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
              max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.01, precision="bf16")
rep.upload_dataset(ds)
lib = rep.lib
buf = np.zeros((16384, 3), np.int64)
for k in range(3):
    lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
    rep.load_batch_stream(k * cfg.b_max, cfg.b_max); rep.train_step(False); torch.cuda.synchronize()
n = lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
ev = buf[:n]
roles, cur = [], [ev[0]]
for e in ev[1:]:
    if e[0] < cur[-1][0]:
        roles.append(cur); cur = []
    cur.append(e)
roles.append(cur)
t0 = min(int(r[0][0]) for r in roles)
for i, r in enumerate(roles):
    print("role %d: %d events, first +%d last +%d" % (i, len(r), r[0][0] - t0, r[-1][0] - t0))
    print("   " + " ".join("%d:%d@%d" % (int(c), int(tile), int(t - t0)) for t, c, tile in r[:400]))
