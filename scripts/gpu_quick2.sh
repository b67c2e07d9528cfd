mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error" gpurun_out/t_gpu.log | tail -3
bash scripts/x_probe.sh
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 120 python scripts/trace_stats.py 2>&1 | tail -60 > gpurun_out/trace_stats.log
