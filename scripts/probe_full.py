"""Step-by-step probe of the full-size path with timings (debug aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen
from paper_2110_07029_b200.api import Replica
name = sys.argv[1] if len(sys.argv) > 1 else "amazon670k"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
cfg = synthgen.CONFIGS[name]
t = time.time(); ds = synthgen.make_dataset(cfg, n=n); print("gen", time.time() - t, flush=True)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
              max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.1, precision="bf16")
rep.upload_dataset(ds); torch.cuda.synchronize(); print("init+upload ok", flush=True)
lib = rep.lib
import ctypes as C
lib.as_profile(rep.ctx, 1)
for k in range(3):
    t = time.time(); rep.load_batch_stream(k * 1024, 1024); l = rep.train_step(True); print("step", k, "loss", l, "s", time.time() - t, flush=True)
ms = (C.c_double * 8)(); calls = (C.c_int64 * 8)(); nl = C.c_int64()
lib.as_profile_read(rep.ctx, ms, calls, C.byref(nl))
print("phases ms", [round(ms[i] / max(1, calls[i]), 4) for i in range(8)], "launches", nl.value, flush=True)
t = time.time()
for k in range(20):
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False)
torch.cuda.synchronize(); print("20 steps s", time.time() - t, flush=True)
t = time.time(); a = rep.merge([20], [1024]); torch.cuda.synchronize(); print("merge", a, time.time() - t, flush=True)
lib.as_profile_read(rep.ctx, ms, calls, C.byref(nl))
print("phases ms", [round(ms[i] / max(1, calls[i]), 4) for i in range(8)], flush=True)
