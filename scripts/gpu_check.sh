mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "rescale" > gpurun_out/t_resc.log 2>&1; echo "rescale tests rc=$?"; tail -3 gpurun_out/t_resc.log
timeout -s KILL 150 python scripts/probe_bench.py 490449 > gpurun_out/pb1.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/pb1.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --verbose > gpurun_out/bench1.log 2>gpurun_out/bench1.err; echo "bench rc=$?"; tail -5 gpurun_out/bench1.err; tail -3 gpurun_out/bench1.log
