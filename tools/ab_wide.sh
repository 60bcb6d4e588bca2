mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --config wide10 --steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline"
for i in 1 2; do
  timeout 300 $B > gpurun_out/ab_new_$i.log 2>&1
  DASH_LIB_PATH=paper_2305_18376_b200/libdash_b200_old.so timeout 300 $B > gpurun_out/ab_old_$i.log 2>&1
done
exit 0
