# GPU tests (R14 literal merges) + exp split A/B (1 exp in 2 / 3 / 4 on the FMA pipe)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
PARITY_LOG=gpurun_out/parity_errors_ze.json timeout -s KILL 900 python -m pytest tests/ -q -m gpu > gpurun_out/t_gpu_ze.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_ze.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazon670k
