mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
for rep in 1 2; do for v in libadasgd_x_nofold libadasgd_x_nofold3 libadasgd; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_fold3.log
