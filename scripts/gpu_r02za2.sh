# quick default bench (JSON line check); heterogeneous replay at the WikiLSHTC-325K and Delicious-200K
# shapes with two ranks sharing the one GPU (functional: routing, Alg. 1 batch sizes, Alg. 2 weights)
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-spmm-sweep --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_quick.log 2>&1; echo "quick rc=$?"; tail -c 400 gpurun_out/bench_quick.log
timeout -s KILL 900 python bench.py --gpus 2 --config wikilshtc325k --hetero --steps 3 --warmup 1 --no-spmm-sweep --e2e-steps 1 > gpurun_out/bench_wiki_g2_hetero.log 2> gpurun_out/bench_wiki_g2_hetero.err; echo "wiki rc=$?"; tail -c 900 gpurun_out/bench_wiki_g2_hetero.log
timeout -s KILL 900 python bench.py --gpus 2 --config delicious200k --hetero --steps 2 --warmup 1 --no-spmm-sweep --e2e-steps 1 > gpurun_out/bench_del_g2_hetero.log 2> gpurun_out/bench_del_g2_hetero.err; echo "del rc=$?"; tail -c 900 gpurun_out/bench_del_g2_hetero.log
