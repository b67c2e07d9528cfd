# A/B: pass-1 per-warp b2 (no named barrier); h = 256 update prefetch (AmazonCat); parity
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/t_gpu_z.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_z.log
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazon670k
bash scripts/x_probe.sh amazoncat13k
