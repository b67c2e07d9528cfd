# round-end style run: all GPU tests, smoke, bench (+cpu baseline), reference arm,
# ncu launch list of the bench command, ncu --set full of the top kernels
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout -s KILL 1200 python -m pytest tests/ -q -x -m gpu --durations=8 > gpurun_out/t_gpu_full.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|error" gpurun_out/t_gpu_full.log | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.log 2>gpurun_out/bench_full.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1400 -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm-sweep --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_out_|k_seg_bulk|k_combine|k_label|k_tr_" -s 14 -c 14 -o gpurun_out/prof_final -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_final.log 2>&1; echo "full rc=$?"
