# the N = 2 bench path end to end on one GPU (validation knob, not a measurement): both ranks on device 0, gloo for the F/G sums
mkdir -p gpurun_out
DASH_BENCH_DEVICE=0 DASH_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/n2.log 2>&1; echo "rc=$?" >> gpurun_out/n2.log
DASH_BENCH_DEVICE=0 DASH_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/n2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/n2_ref.log
( time python bench.py > gpurun_out/bench_full.log 2>&1 ) 2> gpurun_out/bench_full_time.log
exit 0
