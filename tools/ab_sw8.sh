mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or config or fullsize or indefinite" > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
Q="--steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline --dropin-steps 0 --no-als --parity-steps 0"
for i in 1 2 3; do
for c in wide64 wide32; do
  python bench.py --config $c $Q > gpurun_out/sw_new_${c}_$i.log 2>&1
  DASH_LIB_PATH=$PWD/paper_2305_18376_b200/libdash_ab_old.so python bench.py --config $c $Q > gpurun_out/sw_old_${c}_$i.log 2>&1
done
done
exit 0
