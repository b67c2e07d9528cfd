export ADASGD_NO_BUILD=1
timeout -s KILL 60 python scripts/tc_bench.py
