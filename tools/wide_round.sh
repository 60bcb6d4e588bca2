mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${WIDE_CONFIGS:-wide10 wide32 wide64}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 4 --cpu-steps 1 > gpurun_out/cfg_$c.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_$c.log
done
exit 0
