mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or config or fullsize or ill" > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
for c in wide32 wide64; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline > gpurun_out/w_$c.log 2>&1; echo "rc=$?" >> gpurun_out/w_$c.log
done
exit 0
