"""Replays bench.py's sequence with a log line after every call (debug aid)."""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen
from paper_2110_07029_b200 import driver
from paper_2110_07029_b200.api import Replica
T0 = time.time()
def log(*a): print("[%.2f]" % (time.time() - T0), *a, flush=True)
cfg = synthgen.CONFIGS["amazon670k"]
ds = synthgen.make_dataset(cfg, n=int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
stream = torch.cuda.Stream()
rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=cfg.b_min, beta=cfg.beta, megabatch=cfg.megabatch,
              max_row_nnz=int(np.diff(ds.row_ptr).max()), max_row_labels=int(np.diff(ds.lab_ptr).max()),
              lr0=0.1, precision="bf16", stream=stream)
rep.upload_dataset(ds); log("ready")
state = driver.ReplayState(1, cfg.b_max, cfg.b_min, cfg.beta, 0.1, synthgen.make_cost_models(1, False))
prof = len(sys.argv) > 2
if prof:
    rep.lib.as_profile(rep.ctx, 1)
pos = 0
for mb in range(6):
    log_, u, _ = state.route(ds.row_ptr, ds.n, pos, cfg.megabatch)
    log("mb", mb, "routed", len(log_), "batches; first", log_[0], "last", log_[-1])
    for k, (i, s, r) in enumerate(log_):
        rep.load_batch_stream(pos + s, r)
        rep.train_step(False)
        if k % 25 == 0:
            torch.cuda.synchronize(); log("  step", k, "ok")
    torch.cuda.synchronize(); log("mb", mb, "steps done")
    rep.merge(u, list(state.b), want_alpha=False); torch.cuda.synchronize(); log("merged")
    state.rescale(u); rep.set_batch_sizes(state.b, state.lr)
    pos += cfg.megabatch
log("done")
