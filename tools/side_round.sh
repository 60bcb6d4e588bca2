mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-fp32 --e2e-steps 4 --no-als --dropin-steps 0 > gpurun_out/bench_side.log 2>&1; echo "rc=$?" >> gpurun_out/bench_side.log
DASH_NO_SIDE_PLAN=1 timeout 900 python bench.py --no-fp32 --e2e-steps 0 --no-als --dropin-steps 0 --parity-steps 0 --no-cpu-baseline > gpurun_out/bench_noside.log 2>&1; echo "rc=$?" >> gpurun_out/bench_noside.log
for c in medium daily; do python tools/small_probe.py $c > gpurun_out/small_$c.log 2>&1; done
exit 0
