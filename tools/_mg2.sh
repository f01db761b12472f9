N=$1
P=29611
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P "$@"; P=$((P+1)); }
run tools/dist_check.py --quick --scale --qft34 > gpurun_out/mgc${N}.log 2>&1; echo rc=$? >> gpurun_out/mgc${N}.log
run bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/mg${N}_qft.log 2>&1
run bench.py --gpus $N --steps 20 --warmup 5 --workload qft34 > gpurun_out/mg${N}_qft34.log 2>&1
