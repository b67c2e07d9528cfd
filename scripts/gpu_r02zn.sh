# pass-1 ring (S^T in 64-class halves, next block's half 0 during this block's half 1): parity + A/B
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zn.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_zn.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh delicious200k
