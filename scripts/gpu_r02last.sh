# last check of the committed state: every GPU test, smoke, default bench
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
PARITY_LOG=gpurun_out/parity_errors_last.json timeout -s KILL 1500 python -m pytest tests/ -q -m gpu > gpurun_out/t_gpu_last.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_last.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 1200 python bench.py > gpurun_out/bench_last.log 2> gpurun_out/bench_last.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_last.log
