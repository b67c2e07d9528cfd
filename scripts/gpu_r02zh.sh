# h = 256 last-block update through the H stages (LASTSMEM): parity + AmazonCat A/B
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zh.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zh.log
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazoncat13k
