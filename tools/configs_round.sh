# every BASELINE config shape through bench.py (1 GPU): device-resident latency, e2e, CPU oracle
mkdir -p gpurun_out
for c in medium daily wide10 wide32 wide64; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 4 --cpu-steps 1 > gpurun_out/cfg_$c.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_$c.log
done
exit 0
