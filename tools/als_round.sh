mkdir -p gpurun_out
for c in medium daily; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/als_launches_$c.csv python tools/als_probe.py $c 2 > gpurun_out/als_$c.log 2>&1
done
exit 0
