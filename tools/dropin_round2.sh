mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/als_order_probe.py medium daily daily > gpurun_out/als_order.log 2>&1
python tools/als_order_probe.py daily medium daily >> gpurun_out/als_order.log 2>&1
timeout 900 python bench.py --no-fp32 --e2e-steps 0 --no-als --parity-steps 0 --no-cpu-baseline --steps 5 --dropin-steps 4 > gpurun_out/bench_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dropin.log
exit 0
