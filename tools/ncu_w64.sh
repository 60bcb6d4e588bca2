mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slicesw -s 3 -c 1 -o gpurun_out/w64_full python bench.py --config wide64 --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu_w64.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_w64.log
exit 0
