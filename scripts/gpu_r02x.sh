# A/B: S0POLL (decoupled S issue), REGS3 (softmax 160 regs), LATEMK; parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_x.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_x.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazon670k
