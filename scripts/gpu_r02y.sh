# AmazonCat-13K / WikiLSHTC-325K kernel durations (ncu launch list) and full captures of the sparse kernels + h=256 passes
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for cfg in amazoncat13k wikilshtc325k; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_$cfg.csv python scripts/probe_full.py $cfg 60000 > gpurun_out/ncu_list_$cfg.log 2>&1; echo "list $cfg rc=$?"
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_out_|k_seg_bulk|k_combine" -s 20 -c 6 -o gpurun_out/prof_cat -f python scripts/probe_full.py amazoncat13k 60000 > gpurun_out/ncu_cat.log 2>&1; echo "full cat rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_seg_bulk" -s 4 -c 2 -o gpurun_out/prof_wiki -f python scripts/probe_full.py wikilshtc325k 60000 > gpurun_out/ncu_wiki.log 2>&1; echo "full wiki rc=$?"
timeout -s KILL 300 python scripts/x_probe.py amazoncat13k; timeout -s KILL 300 python scripts/x_probe.py wikilshtc325k; timeout -s KILL 300 python scripts/x_probe.py delicious200k
