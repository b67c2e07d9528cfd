mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_out_bwd -s 3 -c 1 -o gpurun_out/prof_bwd -f python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_bwd.log 2>&1; echo "bwd rc=$?"
