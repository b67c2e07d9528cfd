"""Run a few full-size steps on the trace build and print the pass-2 event log of CTA 0."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen
from paper_2110_07029_b200 import _lib as L
from paper_2110_07029_b200.api import Replica
cfg = synthgen.CONFIGS["amazon670k"]
ds = synthgen.make_dataset(cfg, n=20000)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
              max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.1, precision="bf16")
rep.upload_dataset(ds)
lib = rep.lib
buf = np.zeros((16384, 3), np.int64)
for k in range(3):
    lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False); torch.cuda.synchronize()
n = lib.as_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_int64)), 16384)
names = {1: "mma wait_p", 2: "mma got_p", 3: "mma wait_h", 4: "mma got_h", 5: "mma got_h/issue_S",
         6: "smx wait_s", 7: "smx got_s", 8: "smx computed", 9: "smx got_gempty", 10: "prod load_h",
         11: "upd wait_dw", 12: "upd got_dw", 13: "upd rmw done", 14: "upd block done"}
ev = sorted(buf[:n].tolist())
t0 = ev[0][0]
prev = t0
sel = ev[len(ev)//3: len(ev)//3 + 120]
t0 = sel[0][0]; prev = t0
for t, c, tile in sel:
    if True:
        print("%8d %+7d  %-16s %d" % (t - t0, t - prev, names.get(c, c), tile))
        prev = t
