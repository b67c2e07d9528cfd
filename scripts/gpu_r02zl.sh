# transposes' fork point / priority (AmazonCat-13K, Amazon-670K); W2S bf16 shadow by TMA; parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zl.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zl.log
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazon670k
