mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/t_gpu.log | grep -E "passed|failed|Error|assert"
timeout -s KILL 150 python scripts/probe_full.py amazon670k 60000 > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; tail -4 gpurun_out/probe.log
