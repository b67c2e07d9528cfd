# pass-2 role trace of CTA 0 (build: python paper_2110_07029_b200/build.py --trace)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 120 python scripts/trace_stats.py 2>&1 | tail -40 > gpurun_out/trace_stats.log
