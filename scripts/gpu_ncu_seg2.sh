mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_small.csv python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_small.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_seg_bulk" -s 10 -c 4 -o gpurun_out/prof_segbulk -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_sparse.log 2>&1; echo "sparse rc=$?"
