mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
P=paper_2110_07029_b200
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step_parity or full_size_amazon670k_sampled or label_heavy or rescale or deterministic or empty or grid" > gpurun_out/t_gpu_r02j.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_gpu_r02j.log
ADASGD_LIB=$PWD/$P/libadasgd_x_nofold.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "one_step_parity or full_size_amazon670k_sampled" > gpurun_out/t_gpu_r02j_nofold.log 2>&1; echo "tests nofold rc=$?"; tail -2 gpurun_out/t_gpu_r02j_nofold.log
for rep in 1 2; do for v in libadasgd_x_full libadasgd libadasgd_x_nofold libadasgd_x_nofold6; do
  ADASGD_LIB=$PWD/$P/$v.so timeout -s KILL 120 python scripts/x_probe.py amazon670k 2>&1 | tail -1
done; done | tee gpurun_out/x_probe_half.log
