mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_out_" -s 6 -c 2 -o gpurun_out/prof_tc2 -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_tc2.log 2>&1; echo "tc rc=$?"
