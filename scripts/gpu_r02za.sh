# A/B: combine with all partials loaded up front (COMBINE_MAXS=24 vs 1)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_za.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_za.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazoncat13k
