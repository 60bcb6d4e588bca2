mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in medium daily; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/als_launches_$c.csv python tools/als_probe.py $c 2 > gpurun_out/als_$c.log 2>&1
python tools/als_probe.py $c 3 > gpurun_out/als_t_$c.log 2>&1
done
exit 0
