# sparse-kernel shapes at h = 128: Amazon-670K, WikiLSHTC-325K, Delicious-200K
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for c in amazon670k wikilshtc325k delicious200k; do bash scripts/x_probe.sh $c; done
for c in wikilshtc325k delicious200k; do bash scripts/x_probe.sh $c; done
