#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   1. plain bench line, 2. ncu launch list of the same command (cold, serialised),
#   3. one `--set full` capture of each hot kernel (after 3 warm-up steps).
set -u
TAG=${1:-r01}
KERNELS=${2:-"k_slices3 k_big k_xv3 k_fgemm3"}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_ncu_list.log 2>&1
echo "launch list rc=$?"
for k in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 3 --launch-count 1 \
      -o $OUT/${TAG}_full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > $OUT/${TAG}_ncu_full_$k.log 2>&1
  echo "full $k rc=$?"
done
