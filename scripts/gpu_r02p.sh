mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=$PWD/paper_2110_07029_b200
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step_parity or full_size_amazon670k_sampled or label_heavy or deterministic or grid" > gpurun_out/t_gpu_r02p.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02p.log
for rep in 1 2 3; do for v in libadasgd_x_prevfull libadasgd libadasgd_x_nosoft; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_fetch.log
