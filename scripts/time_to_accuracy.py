"""Synthetic time-to-accuracy harness (the paper's
methodology: top-1 accuracy on the test set after every mega-batch).

Adaptive SGD vs the comparison methods (R26: elastic model averaging, gradient
aggregation) on ONE GPU holding N replicas (local-group merge), under the same
heterogeneous replay (per-replica slowdowns 1.00-1.32).  Time axis = the
replayed makespan (sum over mega-batches of max_i t_i, the straggler-bound
wall time the replay models) plus the measured device time.  The data are a
planted-signal synthetic XML set (synthgen.make_planted_dataset): accuracy
numbers here say nothing about the paper's datasets.

    python scripts/time_to_accuracy.py [N] [megabatches] > gpurun_out/tta.jsonl
"""
import json
import os
import re
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthgen
from paper_2110_07029_b200 import driver
from paper_2110_07029_b200.api import Replica, group_merge

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
MB = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = synthgen.XMLConfig("tta", 20000, 2000, 48000, 30.0, 3.0, 128, 256, 1, 77)
full = synthgen.make_planted_dataset(cfg)
train = full.rows(np.arange(40000))
test = full.rows(np.arange(40000, 48000))
p0 = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
costs = synthgen.make_cost_models(N, hetero=True)
lr0 = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
ALGOS = sys.argv[4].split(",") if len(sys.argv) > 4 else ["adaptive", "adaptive_np", "elastic", "sync"]
b_max, b_min = cfg.b_max, cfg.b_max // 8
for name in ALGOS:
    # "adaptive_np": Adaptive SGD with the perturbation disabled (pert_thr = 0):
    # with the literal ||w||_2 / P metric (R15) perturbation fires at every
    # merge and sum(alpha) = 1 + delta (alpha_r - alpha_s) > 1 inflates the model
    algo = "adaptive" if name.startswith("adaptive") else name
    # "..._sfK": adaptive scaling frequency (R27) with p_max = K
    pert_thr = 0.0 if name.startswith("adaptive_np") else 0.1
    pmax = int(re.search(r"_sf(\d+)", name).group(1)) if "_sf" in name else 1
    # "..._bK": Alg. 1 scaling parameter beta = K (P:274 / Fig. 10b: b_min / 2 and
    # one smaller and one larger value); default b_min / 2
    mb = re.search(r"_b(\d+)", name)
    beta = int(mb.group(1)) if mb else b_min // 2
    M = N * b_max if algo == "sync" else 20 * b_max       # sync: one batch per replica per merge
    gamma = 0.9 if algo == "adaptive" else 0.0
    # "..._gK": momentum gamma = K / 100 of the merge (Alg. 2 line 11)
    mg = re.search(r"_g(\d+)", name)
    if mg:
        gamma = int(mg.group(1)) / 100.0
    reps = [Replica(cfg.d, cfg.C, cfg.h, b_max, p0, b_min=b_min, beta=beta, megabatch=M,
                    max_row_nnz=int(np.diff(full.row_ptr).max()), max_row_labels=int(np.diff(full.lab_ptr).max()),
                    lr0=lr0, gamma=gamma, pert_thr=pert_thr, precision="bf16", rank=i, world=N, algo=algo)
            for i in range(N)]
    st = driver.ReplayState(N, b_max, b_min, beta, lr0, costs, algo=algo, scale_pmax=pmax)
    for r in reps:
        r.upload_dataset(train)
    n = len(train.row_ptr) - 1
    sim_ps, gpu_s, seen = 0, 0.0, 0
    total = MB * 20 * b_max                                # same samples for every method
    while seen < total:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pos = seen % n
        log, u, clocks = st.route(train.row_ptr, n, pos, M)
        for (i, start, rows) in log:
            reps[i].load_batch_stream(pos + start, rows)
            reps[i].train_step(False)
        b_used = list(st.b)
        group_merge(reps, u, b_used)
        st.rescale(u)
        for r in reps:
            r.set_batch_sizes(st.b, st.lr)
        torch.cuda.synchronize()
        gpu_s += time.perf_counter() - t0
        sim_ps += max(clocks)
        seen += M
        if seen % (20 * b_max) and seen < total:
            continue
        acc = reps[0].evaluate(test)                   # replicas restart from wbar
        print(json.dumps({"algo": name, "lr0": lr0, "samples": seen, "replay_s": sim_ps * 1e-12, "gpu_s": round(gpu_s, 4),
                          "top1": acc, "u": u, "b": b_used, "period": st.period}), flush=True)
    for r in reps:
        r.close()
    torch.cuda.empty_cache()
