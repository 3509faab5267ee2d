cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
for a in "--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er" "--config 2 --op er"; do
  timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 >> gpurun_out/g1_kernels.txt
done
CMD="python tools/bench_kernel.py --config 3 --op er --reps 3"
timeout 300 $CMD > gpurun_out/g1_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_assemble -s 2 -c 1 -o gpurun_out/g1_c3er $CMD > gpurun_out/g1_ncu.log 2>&1; echo ncu=$? >> gpurun_out/g1_kernels.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g1_pytest.log 2>&1; echo pytest=$? >> gpurun_out/g1_kernels.txt
