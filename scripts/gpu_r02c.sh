mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
for rep in 1 2; do for v in libadasgd_x_oldupd libadasgd libadasgd_x_updpipe; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_upd.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "merge_weighted or one_step_parity or full_size_amazon670k_sampled" > gpurun_out/t_gpu_r02c.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_gpu_r02c.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_r02c.log 2>gpurun_out/bench_r02c.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_r02c.log; tail -3 gpurun_out/bench_r02c.err
