P=29961
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P "${@:2}"; P=$((P+1)); }
run 4 bench.py --gpus 4 --steps 20 --warmup 5 --workload qft34 > gpurun_out/if_qft34.log 2>&1
run 4 bench.py --gpus 4 --steps 3 --warmup 3 --workload qv > gpurun_out/if_qv.log 2>&1
true
