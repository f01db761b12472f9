N=$1
P=29511
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; P=$((P+1)); }
run --steps 20 --warmup 5 > gpurun_out/mg${N}_qft.log 2>&1
run --steps 3 --warmup 3 --workload qv > gpurun_out/mg${N}_qv.log 2>&1
run --steps 20 --warmup 5 --workload qft34 > gpurun_out/mg${N}_qft34.log 2>&1
[ "$N" -ge 4 ] && run --steps 3 --warmup 3 --workload qaoa > gpurun_out/mg${N}_qaoa.log 2>&1
