mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-fp32 --e2e-steps 0 --no-als --parity-steps 0 --no-cpu-baseline --dropin-steps 0 --steps 10 > gpurun_out/bench_fit.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fit.log
for c in medium wide10 wide64; do timeout 600 python bench.py --config $c --no-fp32 --e2e-steps 0 --no-als --parity-steps 0 --no-cpu-baseline --dropin-steps 0 --steps 10 --warmup 3 > gpurun_out/bench_fit_$c.log 2>&1; done
exit 0
