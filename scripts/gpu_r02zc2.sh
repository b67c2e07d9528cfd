# synthetic time-to-accuracy: Alg. 1 beta sweep (b_min / 4, b_min / 2 (paper default), b_min, 2 b_min), 4 replicas, heterogeneous replay
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 1800 python scripts/time_to_accuracy.py 4 60 1.0 adaptive_np_b8,adaptive_np_b16,adaptive_np_b32,adaptive_np_b64 > gpurun_out/tta_beta.jsonl 2> gpurun_out/tta_beta.err; echo "tta rc=$?"; tail -4 gpurun_out/tta_beta.jsonl | cut -c1-300
