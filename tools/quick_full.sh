mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in wide32 wide64; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline --dropin-steps 0 --no-als --parity-steps 0 > gpurun_out/w_$c.log 2>&1
done
exit 0
