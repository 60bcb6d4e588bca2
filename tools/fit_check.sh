mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py tests/test_gpu_fp32.py tests/test_gpu_als.py tests/test_gpu_history.py -m gpu -x -q > gpurun_out/pytest_fit.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fit.log
for c in large medium wide10 wide64; do timeout 600 python bench.py --config $c --no-fp32 --e2e-steps 0 --no-als --parity-steps 1 --no-cpu-baseline --dropin-steps 0 --steps 5 --warmup 3 > gpurun_out/bench_fit_$c.log 2>&1; done
exit 0
