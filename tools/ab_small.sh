mkdir -p gpurun_out
for i in 1 2; do
for c in medium daily; do
  python tools/small_probe.py $c 120 > gpurun_out/ab_small_${c}_bigx_$i.log 2>&1
  DASH_NO_BIGX=1 python tools/small_probe.py $c 120 > gpurun_out/ab_small_${c}_nobigx_$i.log 2>&1
done
done
exit 0
