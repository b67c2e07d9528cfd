# sparse-kernel shapes at h = 256 (AmazonCat-13K): warps / stages / group size
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazoncat13k
