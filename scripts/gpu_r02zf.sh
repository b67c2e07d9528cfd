# AmazonCat-13K (h = 256) pass 1 / pass 2 / combine full captures after the round-2 changes
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_out_|k_combine|k_seg_bulk" -s 20 -c 5 -o gpurun_out/prof_cat2 -f python scripts/probe_full.py amazoncat13k 60000 > gpurun_out/ncu_cat2.log 2>&1; echo "full cat rc=$?"
