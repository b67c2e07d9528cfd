mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_r02l.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_gpu_r02l.log
for rep in 1 2; do for v in libadasgd_x_norot libadasgd; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_rot.log
timeout -s KILL 900 python bench.py --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_r02l.log 2>gpurun_out/bench_r02l.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02l.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'])"
