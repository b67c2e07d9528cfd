"""Tiny-shape run of every step kernel for compute-sanitizer (tools only):
one bf16 step (tcgen05 passes 1 and 2, SpMM, transposes, combine, dW1), one
fp32 step, a top-1 evaluation and a merge, on a 2-row-tile batch with a
ragged tail and C % 128 != 0."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthgen
from paper_2110_07029_b200.api import Replica

cfg = synthgen.XMLConfig("san", 2000, 1000, 400, 20.0, 3.0, 128, 256, 1, 3)
ds = synthgen.make_dataset(cfg, n=400)
p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, 5)
sub = ds.rows(np.arange(200))
for prec in ("bf16", "fp32"):
    rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                  max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.5, precision=prec, debug_grads=True)
    rep.load_batch_csr(200, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    print(prec, "loss", rep.train_step(want_loss=True), flush=True)
    top, hits = rep.eval_top1(200, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    rep.merge_weighted([0.7])
    rep.merge([3], [256])
    rep.close()
print("sanitize probe done", flush=True)
