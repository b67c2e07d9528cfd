mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
timeout -s KILL 120 python scripts/nccl_premul_probe.py > gpurun_out/nccl_premul.log 2>&1; cat gpurun_out/nccl_premul.log | tail -8
for v in libadasgd libadasgd_x_noexp libadasgd_x_nosoft libadasgd_x_noupd libadasgd_x_emu0 libadasgd_x_emu2 libadasgd_x_nomma2 libadasgd_x_nomma1 libadasgd; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done | tee gpurun_out/x_probe_decomp.log
