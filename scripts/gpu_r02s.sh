mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_r02s.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02s.log
for rep in 1 2 3; do
  ADASGD_NO_SLICE=1 timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/gather /'
  timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/slice  /'
done | tee gpurun_out/x_probe_slice.log
