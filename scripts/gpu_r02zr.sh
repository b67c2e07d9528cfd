# exp split in the real passes: 1 in 3 (product), 1 in 4, 1 in 6, none (all MUFU)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for k in 1 2; do bash scripts/x_probe.sh amazon670k; done
