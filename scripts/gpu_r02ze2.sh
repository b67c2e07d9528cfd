# synthetic time-to-accuracy by replica count (N = 1, 2, 4, 8), adaptive (perturbation off) vs elastic averaging
mkdir -p gpurun_out
export ADASGD_NO_BUILD=1
for N in 1 2 4 8; do
  timeout -s KILL 900 python scripts/time_to_accuracy.py $N 60 1.0 adaptive_np > gpurun_out/tta_n${N}_adaptive.jsonl 2> gpurun_out/tta_n${N}.err; echo "N=$N adaptive rc=$?"
  timeout -s KILL 900 python scripts/time_to_accuracy.py $N 60 4.0 elastic > gpurun_out/tta_n${N}_elastic.jsonl 2>> gpurun_out/tta_n${N}.err; echo "N=$N elastic rc=$?"
done
