mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "top1 or sparse_long" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error|assert|rel err" gpurun_out/t_gpu.log | tail -8
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2> gpurun_out/bench3.err; echo bench rc=$?; tail -c 600 gpurun_out/bench3.err
