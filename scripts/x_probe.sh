# time every experiment build (paper_2110_07029_b200/libadasgd_x_*.so) + the product build
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
cfgname=${1:-amazon670k}
for lib in paper_2110_07029_b200/libadasgd.so $(ls paper_2110_07029_b200/libadasgd_x_*.so 2>/dev/null); do
  ADASGD_LIB=$PWD/$lib timeout -s KILL 120 python scripts/x_probe.py $cfgname 2>&1 | tail -1
done | tee gpurun_out/x_probe.log
