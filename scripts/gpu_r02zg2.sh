# pass 1 W stages 3 / 4 (product) / 5
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for k in 1 2 3; do timeout -s KILL 300 bash scripts/x_probe.sh amazon670k; done
