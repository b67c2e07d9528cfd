"""Per-phase timing of the step for experiment builds (ADASGD_LIB=...); tools only."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen
from paper_2110_07029_b200.api import Replica
from paper_2110_07029_b200 import _lib as L

cfg = synthgen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "amazon670k"]
ds = synthgen.make_dataset(cfg, n=40000)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
              max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.01, precision="bf16", stream=torch.cuda.Stream(priority=-1))
rep.upload_dataset(ds)
for k in range(3):
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(rep.stream)
for k in range(30):
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False)
e1.record(rep.stream)
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1) / 30
rep.lib.as_profile(rep.ctx, 1)
for k in range(30):
    rep.load_batch_stream(k * 1024, 1024); rep.train_step(False)
torch.cuda.synchronize()
ms = (C.c_double * 8)(); calls = (C.c_int64 * 8)(); nl = C.c_int64()
rep.lib.as_profile_read(rep.ctx, ms, calls, C.byref(nl))
print("%-40s" % os.path.basename(os.environ.get("ADASGD_LIB", "libadasgd.so")),
      "step=%.4f" % step_ms, " ".join("%s=%.4f" % (L.AS_PH_NAMES[i], ms[i] / max(1, calls[i])) for i in range(7)), flush=True)
