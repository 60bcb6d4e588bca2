mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in medium daily; do python tools/small_probe.py $c > gpurun_out/small_$c.log 2>&1; done
python tools/host_small.py 2>&1 | head -n 3 > gpurun_out/host_small.log
exit 0
