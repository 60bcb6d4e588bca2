# wide configs after the wide-J GEMMs: parity, bench, then an ncu --set full capture of k_slicesw<8> (wide64)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py -m gpu -x -q -k "wide or config or fullsize" > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
for c in wide32 wide64; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline > gpurun_out/w_$c.log 2>&1; echo "rc=$?" >> gpurun_out/w_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slicesw -s 3 -c 1 -o gpurun_out/w64_full python bench.py --config wide64 --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu_w64.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_w64.log
exit 0
