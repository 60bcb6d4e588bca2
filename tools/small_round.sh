mkdir -p gpurun_out
for c in medium daily; do
  python tools/small_probe.py $c > gpurun_out/small_$c.log 2>&1
  DASH_HOST_TIMING=1 python tools/small_probe.py $c 24 2>&1 | tail -n 12 >> gpurun_out/small_$c.log
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 60 --csv --log-file gpurun_out/small_launches_$c.csv python tools/small_probe.py $c 24 > /dev/null 2>&1
done
exit 0
