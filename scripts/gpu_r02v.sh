# session re-entry: GPU tests, short bench, x_probe, pass-2 source-level ncu capture
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_v.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_v.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_v.log 2>gpurun_out/bench_v.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_v.log
bash scripts/x_probe.sh amazon670k
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_out_bwd|k_out_fwd|k_seg_bulk" -s 6 -c 4 -o gpurun_out/prof_v -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_v.log 2>&1; echo "ncu rc=$?"
