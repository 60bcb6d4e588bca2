mkdir -p gpurun_out
Q="--config wide64 --steps 10 --warmup 3 --no-fp32 --e2e-steps 0 --no-cpu-baseline --dropin-steps 0 --no-als --parity-steps 0"
for i in 1 2 3; do
  python bench.py $Q > gpurun_out/ab_shfl_$i.log 2>&1
  DASH_LIB_PATH=$PWD/paper_2305_18376_b200/libdash_ab_serial.so python bench.py $Q > gpurun_out/ab_serial_$i.log 2>&1
done
exit 0
