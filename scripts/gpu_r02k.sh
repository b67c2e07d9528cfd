# round-2 baseline: tests, smoke, bench, reference arm, ncu launch list + full capture, sanitizers
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
PARITY_LOG=gpurun_out/parity_errors_r02.json timeout -s KILL 1500 python -m pytest tests/ -q -m gpu --durations=8 > gpurun_out/t_gpu_r02k.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_r02k.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_r02k.log 2>gpurun_out/bench_r02k.err; echo "bench rc=$?"; tail -c 200 gpurun_out/bench_r02k.log
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02k.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_r02k.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1400 -c 400 --csv --log-file gpurun_out/launches_r02k.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm-sweep --e2e-steps 1 > gpurun_out/ncu_bench_r02k.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_out_|k_seg_bulk|k_combine|k_label|k_tr_|k_gather" -s 14 -c 16 -o gpurun_out/prof_r02k -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_full_r02k.log 2>&1; echo "full rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
