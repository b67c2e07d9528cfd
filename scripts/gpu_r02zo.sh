# threaded host staging: parity tests, AmazonCat + Amazon-670K bench e2e
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zo.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_zo.log
timeout -s KILL 600 python bench.py --config amazoncat13k --steps 10 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_amazoncat_zo.log 2>gpurun_out/bench_amazoncat_zo.err; echo "bench amazoncat rc=$?"
timeout -s KILL 900 python bench.py --steps 10 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_zo.log 2>gpurun_out/bench_zo.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/bench_amazoncat_zo.log", "gpurun_out/bench_zo.log"]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["roofline"]["frac"])
PY
