mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_r02r.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02r.log
for rep in 1 2 3; do
  ADASGD_LT_SEPARATE=1 timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/ltsep /'
  timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/ltp1  /'
done | tee gpurun_out/x_probe_ltfuse.log
for cfgn in delicious200k wikilshtc325k amazoncat13k; do
  ADASGD_LT_SEPARATE=1 timeout -s KILL 200 python scripts/x_probe.py $cfgn 2>&1 | tail -1 | sed "s/^/ltsep $cfgn /"
  timeout -s KILL 200 python scripts/x_probe.py $cfgn 2>&1 | tail -1 | sed "s/^/ltp1  $cfgn /"
done | tee -a gpurun_out/x_probe_ltfuse.log
