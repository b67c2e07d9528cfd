# same-box A/B: HEAD vs the f2 build (fd9425a) vs the session-start build (a7b9c6a); full-size AmazonCat parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "amazoncat13k" > gpurun_out/t_gpu_zp.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu_zp.log
for k in 1 2 3; do bash scripts/x_probe.sh amazon670k; done
