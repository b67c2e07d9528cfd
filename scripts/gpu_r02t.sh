mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=$PWD/paper_2110_07029_b200
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step or full_size_amazon670k_sampled or deterministic" > gpurun_out/t_gpu_r02t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02t.log
for rep in 1 2 3; do for v in libadasgd_x_nosusp libadasgd; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_susp.log
for v in libadasgd_x_nosusp libadasgd; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 900 python bench.py --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_susp_$v.log 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_susp_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['clocks'])"
done
