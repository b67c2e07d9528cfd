# h = 256 label terms in pass 1's idle warpgroup (6 warps per CTA) vs the separate kernel; parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zk.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zk.log
for k in 1 2; do
timeout -s KILL 120 python scripts/x_probe.py amazoncat13k
ADASGD_LT_SEPARATE=1 timeout -s KILL 120 python scripts/x_probe.py amazoncat13k
done
