mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-fp32 --e2e-steps 0 --no-als --parity-steps 0 --no-cpu-baseline --steps 5 > gpurun_out/bench_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dropin.log
for c in medium daily; do
timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-fp32 --e2e-steps 0 --no-als --parity-steps 0 --no-cpu-baseline > gpurun_out/bench50_$c.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-fp32 --e2e-steps 0 --dropin-steps 0 --parity-steps 0 --no-cpu-baseline > gpurun_out/bench_als.log 2>&1
exit 0
