mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "not top1" > gpurun_out/t_gpu_r02d.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_gpu_r02d.log
for rep in 1 2; do for v in libadasgd_x_oldupd libadasgd_x_noring libadasgd; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_ring.log
ADASGD_LIB=$PWD/$P/libadasgd_trace.so timeout -s KILL 120 python scripts/trace_stats.py > gpurun_out/trace_ring.txt 2>&1; tail -30 gpurun_out/trace_ring.txt
