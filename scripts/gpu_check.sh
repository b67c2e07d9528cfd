mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed" gpurun_out/t_gpu.log | tail -2
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>gpurun_out/bench2.err; echo "bench rc=$?"; tail -1 gpurun_out/bench2.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step','e2e','gpu_launches']}); print(d['roofline']['frac'], d['roofline']['spmm']); print({k:(round(v['ms']/max(1,v['calls']),4)) for k,v in d['phases_ms'].items()})"
