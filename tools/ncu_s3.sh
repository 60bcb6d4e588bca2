mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slices3 -s 6 -c 1 -o gpurun_out/s3_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 --dropin-steps 0 --no-als > gpurun_out/ncu_s3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_s3.log
