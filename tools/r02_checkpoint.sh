# round-2 checkpoint measurement: tests, smoke, default bench, reference arm, launch list, every config,
# ncu --set full captures of the wide-J GEMMs and the wide slice kernel (DRAM traffic per launch)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 --dropin-steps 0 --no-als --parity-steps 0 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
for c in medium daily wide10 wide32 wide64; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fp32 --e2e-steps 4 --cpu-steps 1 --no-als > gpurun_out/cfg_$c.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_$c.log
done
Q="--steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 --dropin-steps 0 --no-als --parity-steps 0"
cap() {  # cap <config> <kernel regex> <tag>: one --set full capture, kept as raw-metric CSV (the .ncu-rep stays on the box)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o /tmp/$3 python bench.py --config $1 $Q > gpurun_out/ncu_$3.log 2>&1
  ncu -i /tmp/$3.ncu-rep --page raw --csv > gpurun_out/ncu_$3_raw.csv 2>/dev/null
  ncu -i /tmp/$3.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$3_src.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/$3_src.csv 40 > gpurun_out/ncu_$3_lines.txt 2>&1
  rm -f /tmp/$3.ncu-rep /tmp/$3_src.csv
}
cap wide10 k_xvw w10_xvw
cap wide10 k_fgemmw w10_fgemmw
cap wide64 k_slicesw w64_slicesw
cap wide64 k_xvw w64_xvw
cap wide64 k_fgemmw w64_fgemmw
exit 0
