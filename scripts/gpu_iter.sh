# quick iteration: GPU parity tests (no slow), experiment timings, traces
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
[ -z "$NOTEST" ] && timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t_gpu.log | tail -5
bash scripts/x_probe.sh
timeout -s KILL 120 python scripts/tc_bench.py 6 7 8 9 10 11 12 13 14 | tee gpurun_out/tc_bench.log
for t in paper_2110_07029_b200/libadasgd_x_tr*.so; do [ -f $t ] && ADASGD_LIB=$PWD/$t timeout -s KILL 120 python scripts/trace_stats.py 2>&1 | tail -40; done | tee gpurun_out/trace_stats.log
