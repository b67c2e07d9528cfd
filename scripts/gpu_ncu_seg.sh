# launch list of a few full-size steps + full captures of the sparse kernels (SpMM / dW1 / transposes)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
bash scripts/x_probe.sh
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 120 --csv --log-file gpurun_out/launches_small.csv python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_small.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_seg_gr|k_tr_" -s 40 -c 10 -o gpurun_out/prof_sparse -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_sparse.log 2>&1; echo "sparse rc=$?"
