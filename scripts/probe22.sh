export BENCH_FORCE_DEVICE=0 BENCH_BACKEND=gloo
for w in gemm allgather batched; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --workload $w --no-e2e > gpurun_out/bench_w2_$w.json 2> gpurun_out/bench_w2_$w.err; echo "$w exit=$?"; cat gpurun_out/bench_w2_$w.json | cut -c1-400; tail -2 gpurun_out/bench_w2_$w.err
done
unset BENCH_FORCE_DEVICE BENCH_BACKEND
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 50 --warmup 3 --no-e2e --no-cpu-baseline | cut -c1-300
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 | cut -c1-300; echo "ref exit=$?"
