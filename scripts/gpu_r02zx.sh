# AmazonCat-13K one-block pass 2 with four 64-row H stages (TR64): parity + A/B + CTA-0 trace
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zx.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zx.log
for k in 1 2; do timeout -s KILL 300 bash scripts/x_probe.sh amazoncat13k; done
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 300 python scripts/trace_timeline.py amazoncat13k > gpurun_out/trace_cat_tr64.txt 2>&1; echo "trace rc=$?"
