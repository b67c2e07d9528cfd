# A/B: ECF (bias out of the exponent) and LATEMK (late bitmap read) in pass 2; parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_w.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_w.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazon670k
