#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   bench.sh TAG list       -> plain bench line + ncu launch list (cold, serialised)
#   bench.sh TAG full K1 K2 -> one `--set full` capture per kernel (after 3 warm-up updates)
set -u
TAG=$1; MODE=$2; shift 2
OUT=gpurun_out
mkdir -p $OUT
if [ "$MODE" = list ]; then
  python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
  echo "bench rc=$?"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 200 --csv \
      --log-file $OUT/${TAG}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 1 > $OUT/${TAG}_ncu_list.log 2>&1
  echo "launch list rc=$?"
else
  for k in "$@"; do
    ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 3 --launch-count 1 \
        -o $OUT/${TAG}_full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 1 \
        > $OUT/${TAG}_ncu_full_$k.log 2>&1
    echo "full $k rc=$?"
  done
fi
