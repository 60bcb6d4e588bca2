# wide-rank (R > 16) kernel check: parity tests, then the wide configs' bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or edge or config_shaped" > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
for c in wide32 wide64 wide10; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp32 --dropin-steps 0 --no-als --e2e-steps 0 > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
exit 0
