# end-of-session measurement: default bench line, launch list, --set full of the small-slice kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slices3 -s 6 -c 1 -o gpurun_out/s3_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu_s3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_s3.log
exit 0
