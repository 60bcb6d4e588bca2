# ncu --set full of the large config's four main kernels (raw metrics CSV + per-line stall attribution)
mkdir -p gpurun_out
Q="--steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 0 --dropin-steps 0 --no-als --parity-steps 0"
cap() {
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 -o /tmp/$2 python bench.py $Q > gpurun_out/ncu_$2.log 2>&1
  ncu -i /tmp/$2.ncu-rep --page raw --csv > gpurun_out/ncu_$2_raw.csv 2>/dev/null
  ncu -i /tmp/$2.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$2_src.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/$2_src.csv 40 > gpurun_out/ncu_$2_lines.txt 2>&1
  rm -f /tmp/$2.ncu-rep /tmp/$2_src.csv
}
cap k_slices3 large_slices3
cap "k_bigx<" large_bigx
cap k_xv3 large_xv3
cap k_fgemm3 large_fgemm3
exit 0
