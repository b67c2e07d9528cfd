# full round-end style check: all GPU tests (incl. slow), smoke, bench with cpu baseline, reference arm
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 1200 python -m pytest tests/ -q -x -m gpu --durations=10 > gpurun_out/t_gpu_full.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|error" gpurun_out/t_gpu_full.log | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_full.log 2>gpurun_out/bench_full.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_full.log
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.log
