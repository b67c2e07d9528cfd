# pass-2 CTA-0 timeline at h = 256 (AmazonCat-13K) on the trace build
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 300 python scripts/trace_timeline.py amazoncat13k > gpurun_out/trace_cat.txt 2>&1; echo "trace rc=$?"
