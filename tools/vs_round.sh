mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
Q="--steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline --dropin-steps 0 --no-als --parity-steps 0"
for i in 1 2; do
for c in wide32 wide64; do
  python bench.py --config $c $Q > gpurun_out/vs_new_${c}_$i.log 2>&1
  DASH_OLD_VSOLVE=1 python bench.py --config $c $Q > gpurun_out/vs_old_${c}_$i.log 2>&1
done
done
exit 0
