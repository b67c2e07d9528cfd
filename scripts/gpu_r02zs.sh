# per-pass exp split: product (pass 1 1-in-6, pass 2 none) vs old (3, 3) vs (4, 0); parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zs.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zs.log
for k in 1 2 3; do bash scripts/x_probe.sh amazon670k; done
bash scripts/x_probe.sh delicious200k
bash scripts/x_probe.sh wikilshtc325k
bash scripts/x_probe.sh amazoncat13k
