mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for t in paper_2110_07029_b200/libadasgd_trace.so paper_2110_07029_b200/libadasgd_x_tr*.so; do ADASGD_LIB=$PWD/$t timeout -s KILL 120 python scripts/trace_stats.py 2>&1 | tail -32; done > gpurun_out/trace_stats.log
