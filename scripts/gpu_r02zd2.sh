# synthetic time-to-accuracy: merge momentum gamma sweep (Alg. 2 line 11), 4 replicas, heterogeneous replay
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 1800 python scripts/time_to_accuracy.py 4 60 1.0 adaptive_np_g0,adaptive_np_g50,adaptive_np_g90,adaptive_np_g99 > gpurun_out/tta_gamma.jsonl 2> gpurun_out/tta_gamma.err; echo "tta rc=$?"; tail -2 gpurun_out/tta_gamma.jsonl | cut -c1-300
