mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
bash scripts/x_probe.sh
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 120 python scripts/trace_stats.py 2>&1 | tail -60 | tee gpurun_out/trace_stats.log
