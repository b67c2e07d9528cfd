# re-entry check of HEAD: GPU parity tests + short bench (gpu_check), x_probe of product + variants
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/gpu_check.sh 2>&1 | tail -6
bash scripts/x_probe.sh
