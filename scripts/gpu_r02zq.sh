# softmax instruction-mix throughput vs warps per sub-partition (tools/ubench_softmax.cu)
mkdir -p gpurun_out
timeout -s KILL 120 ./tools/ubench_softmax > gpurun_out/ubench_softmax.txt 2>&1; echo "ubench rc=$?"; cat gpurun_out/ubench_softmax.txt
