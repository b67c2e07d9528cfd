# GPU parity with the seeded random shapes
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
PARITY_LOG=gpurun_out/parity_errors_rand.json timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/t_gpu_rand.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/t_gpu_rand.log
