mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_als.py tests/test_gpu_history.py tests/test_reference_scenarios.py tests/test_checkpoint.py -m gpu -x -q > gpurun_out/pytest_als.log 2>&1; echo rc=$? >> gpurun_out/pytest_als.log
for c in medium daily; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/als_launches_$c.csv python tools/als_probe.py $c 2 > gpurun_out/als_$c.log 2>&1
done
exit 0
