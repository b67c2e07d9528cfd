# quick: GPU parity tests (no full-size), bench, launch list of a few steps
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|Error" gpurun_out/t_gpu.log | tail -3
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>gpurun_out/bench2.err; echo "bench rc=$?"; tail -1 gpurun_out/bench2.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step','gpu_launches']}, 'e2e', round(d['e2e']['value'])); print('tc frac', round(d['roofline']['frac'],4), 'spmm', {k: d['roofline']['spmm'][k] for k in ['achieved','frac']}); print({k:(round(v['ms']/max(1,v['calls']),4)) for k,v in d['phases_ms'].items()})"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 120 --csv --log-file gpurun_out/launches_small.csv python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_small.log 2>&1; echo "launch list rc=$?"
