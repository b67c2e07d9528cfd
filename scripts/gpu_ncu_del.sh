mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_seg_bulk" -s 10 -c 2 -o gpurun_out/prof_seg_del -f python scripts/probe_full.py delicious200k 8192 > gpurun_out/ncu_del.log 2>&1; echo "del rc=$?"
