O=gpurun_out/s6c; mkdir -p $O
VMSPLAT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_2rank.log 2>&1; echo "2-rank rc=$?"
tail -1 $O/bench_2rank.log | cut -c1-600
