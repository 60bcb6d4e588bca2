#!/bin/bash
# one `--set full` capture of kernel $1 (after 3 warm-up steps) -> gpurun_out/$2.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:"$1" --launch-skip 3 --launch-count 1 \
    -o gpurun_out/$2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp32 --e2e-steps 1 > gpurun_out/$2.log 2>&1
echo "ncu $1 rc=$?"
