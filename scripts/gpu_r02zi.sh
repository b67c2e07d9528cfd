# W2S (h = 256, one class block per CTA: W2T block in shared memory, 4 S^T buffers): parity + AmazonCat A/B
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_gpu_zi.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu_zi.log
bash scripts/x_probe.sh amazoncat13k
bash scripts/x_probe.sh amazoncat13k
ADASGD_LIB=$PWD/paper_2110_07029_b200/libadasgd_trace.so timeout -s KILL 300 python scripts/trace_timeline.py amazoncat13k > gpurun_out/trace_cat_w2s.txt 2>&1; echo "trace rc=$?"
