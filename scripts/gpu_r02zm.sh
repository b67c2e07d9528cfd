# full GPU tests after the AmazonCat changes (runtime fork point); AmazonCat + Amazon x_probe
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
PARITY_LOG=gpurun_out/parity_errors_zm.json timeout -s KILL 1200 python -m pytest tests/ -q -m gpu > gpurun_out/t_gpu_zm.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zm.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazon670k
timeout -s KILL 900 python bench.py --config amazoncat13k --steps 10 --no-spmm-sweep --no-cpu-baseline > gpurun_out/bench_amazoncat_zm.log 2>gpurun_out/bench_amazoncat_zm.err; echo "bench amazoncat rc=$?"; tail -c 600 gpurun_out/bench_amazoncat_zm.log
