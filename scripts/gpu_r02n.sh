mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=$PWD/paper_2110_07029_b200
for rep in 1 2; do for v in libadasgd libadasgd_x_notma libadasgd_x_nosoft libadasgd_x_nosoftnoupd libadasgd_x_nosoftnotma libadasgd_x_nosoftnomma1 libadasgd_x_nosoftnomma2; do
  ADASGD_LIB=$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_skeleton.log
