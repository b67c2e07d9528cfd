mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "resident or rank_api or deterministic" > gpurun_out/t_gpu_r02u.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02u.log
for rep in 1 2 3; do
  ADASGD_SLICE_MAIN=1 timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/main /'
  timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1 | sed 's/^/cps  /'
done | tee gpurun_out/x_probe_slicecp.log
for v in 1 0; do
  ADASGD_SLICE_MAIN=$v timeout -s KILL 900 python bench.py --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_slice_$v.log 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_slice_$v.log').read().strip().splitlines()[-1]); print('slice_main=$v', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
