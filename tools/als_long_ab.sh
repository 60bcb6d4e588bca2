mkdir -p gpurun_out
for c in medium daily; do
for L in default 256 512 1024; do
  if [ $L = default ]; then unset DASH_ALS_LONG; else export DASH_ALS_LONG=$L; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_als_polar -c 30 --csv --log-file gpurun_out/alsab_${c}_$L.csv python tools/als_probe.py $c 2 > /dev/null 2>&1
done
done
exit 0
