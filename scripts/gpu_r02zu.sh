# TMEM loads vs a concurrent SS / TS MMA stream (tools/ubench_tmem_mma.cu)
mkdir -p gpurun_out
timeout -s KILL 120 ./tools/ubench_tmem_mma > gpurun_out/ubench_tmem_mma.txt 2>&1; echo "ubench rc=$?"; cat gpurun_out/ubench_tmem_mma.txt
