# A/B of the small-slice kernel across library builds (DASH_LIB_PATH), two runs per arm
mkdir -p gpurun_out
[ -z "$AB_NOTEST" ] && { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; }
B="python bench.py --no-cpu-baseline --no-fp32 --e2e-steps 0 --steps 20 --warmup 5"
for i in 1 2; do
  timeout 300 $B > gpurun_out/ab_new_$i.log 2>&1
  [ -n "$AB_SWEEP" ] && DASH_S3_SWEEP=1 timeout 300 $B > gpurun_out/ab_sweep_$i.log 2>&1
  for v in old a b c; do
    [ -f paper_2305_18376_b200/libdash_b200_$v.so ] && DASH_LIB_PATH=paper_2305_18376_b200/libdash_b200_$v.so timeout 300 $B > gpurun_out/ab_${v}_$i.log 2>&1
  done
done
[ -z "$AB_NONCU" ] && { timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log; }
exit 0
