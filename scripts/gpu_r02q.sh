mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step_parity or full_size_amazon670k_sampled or long_segments or deterministic or empty or resident" > gpurun_out/t_gpu_r02q.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02q.log
for rep in 1 2 3; do
  ADASGD_NO_DW1_FUSE=1 timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/nofuse /'
  timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/fused  /'
done | tee gpurun_out/x_probe_dw1fuse.log
for cfgn in delicious200k wikilshtc325k; do for rep in 1; do
  ADASGD_NO_DW1_FUSE=1 timeout -s KILL 200 python scripts/x_probe.py $cfgn 2>&1 | tail -1 | sed "s/^/nofuse $cfgn /"
  timeout -s KILL 200 python scripts/x_probe.py $cfgn 2>&1 | tail -1 | sed "s/^/fused  $cfgn /"
done; done | tee -a gpurun_out/x_probe_dw1fuse.log
