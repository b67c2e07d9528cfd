# update warps poll their block barriers with nanosleep (not the SYNCS-woken suspend); parity + A/B
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zz.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zz.log
for k in 1 2 3; do timeout -s KILL 300 bash scripts/x_probe.sh amazon670k; done
timeout -s KILL 300 bash scripts/x_probe.sh delicious200k
timeout -s KILL 300 bash scripts/x_probe.sh amazoncat13k
