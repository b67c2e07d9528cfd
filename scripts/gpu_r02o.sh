mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=$PWD/paper_2110_07029_b200
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step_parity or full_size_amazon670k_sampled or label_heavy or rescale or deterministic or empty or grid or merge" > gpurun_out/t_gpu_r02o.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02o.log
for rep in 1 2 3; do for v in libadasgd_x_fullbuf libadasgd libadasgd_x_nosoftfull libadasgd_x_nosoft; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_ping.log
