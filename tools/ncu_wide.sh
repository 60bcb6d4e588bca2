mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slices -s 3 -c 1 -o gpurun_out/w32_full python bench.py --config wide32 --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu_w32.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_w32.log
exit 0
