mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_als_polar_mma -s 2 -c 2 -o /tmp/polar python tools/als_probe.py daily 1 > gpurun_out/ncu_polar.log 2>&1
ncu -i /tmp/polar.ncu-rep --page raw --csv > gpurun_out/ncu_polar_raw.csv 2>/dev/null
ncu -i /tmp/polar.ncu-rep --page source --csv --print-source cuda,sass > /tmp/polar_src.csv 2>/dev/null
python tools/ncu_lines.py /tmp/polar_src.csv 45 > gpurun_out/ncu_polar_lines.txt 2>&1
exit 0
