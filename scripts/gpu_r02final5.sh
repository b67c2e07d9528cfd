# round-2 final (second session, final state): tests, smoke, bench (+AmazonCat, +N=2 on one GPU),
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
PARITY_LOG=gpurun_out/parity_errors_f5.json timeout -s KILL 1500 python -m pytest tests/ -q -m gpu --durations=8 > gpurun_out/t_gpu_f5.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_f5.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f5.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_f5.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_f5.log 2>gpurun_out/bench_f5.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_f5.log
timeout -s KILL 900 python bench.py --config amazoncat13k --steps 10 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_amazoncat_f5.log 2>gpurun_out/bench_amazoncat_f5.err; echo "bench amazoncat rc=$?"
timeout -s KILL 900 python bench.py --gpus 2 --steps 3 --warmup 1 --no-spmm-sweep --e2e-steps 1 > gpurun_out/bench_g2_f5.log 2>gpurun_out/bench_g2_f5.err; echo "bench g2 rc=$?"; tail -c 300 gpurun_out/bench_g2_f5.log
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_f5.log 2>&1; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1400 -c 400 --csv --log-file gpurun_out/launches_f5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm-sweep --e2e-steps 1 > gpurun_out/ncu_bench_f5.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_out_|k_seg_bulk|k_combine|k_label|k_tr_|k_slice|k_gather" -s 12 -c 14 -o gpurun_out/prof_f5 -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_full_f5.log 2>&1; echo "full rc=$?"
