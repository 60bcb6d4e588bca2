# same-box A/B of the wide configs: the working tree's library against paper_2305_18376_b200/libdash_ab_old.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py tests/test_gpu_pdl.py -m gpu -x -q > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
Q="--steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline --dropin-steps 0 --no-als --parity-steps 0"
for i in 1 2 3; do
for c in wide10 wide32 wide64; do
  python bench.py --config $c $Q > gpurun_out/ab_new_${c}_$i.log 2>&1
  DASH_LIB_PATH=$PWD/paper_2305_18376_b200/libdash_ab_old.so python bench.py --config $c $Q > gpurun_out/ab_old_${c}_$i.log 2>&1
done
done
exit 0
