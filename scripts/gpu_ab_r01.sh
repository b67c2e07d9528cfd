# same-box A/B of the round-1 library (commit 8c179e3 sources) against HEAD
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=$PWD/paper_2110_07029_b200
for rep in 1 2 3; do for v in libadasgd_x_r01 libadasgd; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/ab_r01_xprobe.log
for rep in 1 2; do for v in libadasgd_x_r01 libadasgd; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 900 python bench.py --no-spmm-sweep --no-cpu-baseline > gpurun_out/ab_bench_$v.$rep.log 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_bench_$v.$rep.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done; done | tee gpurun_out/ab_r01_bench.log
