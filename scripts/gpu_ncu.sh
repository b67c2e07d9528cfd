mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_out_ -s 4 -c 2 -o gpurun_out/r01_prof_tc -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_tc.log 2>&1; echo "tc rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_seg_chunk -s 2 -c 1 -o gpurun_out/r01_prof_spmm -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_spmm.log 2>&1; echo "spmm rc=$?"
