mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "resident or one_step or empty or invalid" > gpurun_out/t_gpu_r02m.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02m.log
for rep in 1 2; do timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1; done
for rep in 1 2; do timeout -s KILL 900 python bench.py --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_r02m_$rep.log 2>gpurun_out/bench_r02m.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02m_$rep.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"; done
