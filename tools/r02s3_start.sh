# session-3 (round 2) start: tests, smoke, bench, launch list, every config, sanitizer
bash tools/gpu_round.sh
bash tools/configs_round.sh
bash tools/sanitize.sh > gpurun_out/sanitize_summary.log 2>&1
exit 0
