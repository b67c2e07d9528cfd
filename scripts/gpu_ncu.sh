mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 150 --csv --log-file gpurun_out/launches_probe.csv python scripts/probe_full.py amazon670k 60000 > gpurun_out/ncu_probe.log 2>&1; echo "rc=$?"
