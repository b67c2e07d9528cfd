# round 2, first GPU call: full GPU tests (parity log), smoke, mutant sensitivity,
# exp micro-benchmark, short bench
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
PARITY_LOG=gpurun_out/parity_errors_r02.json timeout -s KILL 1500 python -m pytest tests/ -q -m gpu --durations=10 -p no:randomly > gpurun_out/t_gpu_r02a.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/t_gpu_r02a.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for v in p1noo p2nosoft; do
  ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_x_$v.so PARITY_LOG=gpurun_out/parity_mutant_$v.json timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=line -k "(one_step_parity and bf16) or full_size_amazon670k_sampled or rescale" > gpurun_out/t_mutant_$v.log 2>&1; echo "mutant $v rc=$?"; tail -2 gpurun_out/t_mutant_$v.log
done
timeout -s KILL 60 ./tools/ubench_mufu > gpurun_out/ubench_mufu.log 2>&1; cat gpurun_out/ubench_mufu.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_r02a.log 2>gpurun_out/bench_r02a.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_r02a.log
