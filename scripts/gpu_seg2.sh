mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse or one_step or deterministic" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error|assert|rel err" gpurun_out/t_gpu.log | tail -4
bash scripts/x_probe.sh
