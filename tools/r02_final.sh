# round-2 final check of the committed tree: tests, smoke, default bench (the line the driver records), reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 1200 python bench.py > gpurun_out/bench.log 2>&1 ) 2> gpurun_out/bench_time.log; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 --dropin-steps 0 --no-als --parity-steps 0 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
for c in medium daily wide10 wide32 wide64; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 4 --cpu-steps 1 --no-als > gpurun_out/cfg_$c.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_$c.log
done
exit 0
