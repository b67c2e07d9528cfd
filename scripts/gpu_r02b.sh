mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
PARITY_LOG=gpurun_out/parity_errors_r02.json timeout -s KILL 1500 python -m pytest tests/ -q -m gpu --durations=10 > gpurun_out/t_gpu_r02b.log 2>&1; echo "gpu tests rc=$?"; tail -12 gpurun_out/t_gpu_r02b.log
timeout -s KILL 600 python bench.py --gpus 2 --steps 2 --warmup 1 --no-spmm-sweep --e2e-steps 1 > gpurun_out/bench_g2_shared.log 2>gpurun_out/bench_g2_shared.err; echo "bench g2 rc=$?"; tail -c 800 gpurun_out/bench_g2_shared.log; tail -5 gpurun_out/bench_g2_shared.err
timeout -s KILL 900 python bench.py > gpurun_out/bench_r02b.log 2>gpurun_out/bench_r02b.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_r02b.log
