P=29911
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P "${@:2}"; P=$((P+1)); }
N=$1
run $N tools/dist_check.py --quick --scale --qft34 > gpurun_out/mgc${N}.log 2>&1; echo rc=$? >> gpurun_out/mgc${N}.log
run $N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/mg${N}_qft.log 2>&1
run $N bench.py --gpus $N --steps 20 --warmup 5 --workload qft34 > gpurun_out/mg${N}_qft34.log 2>&1
run $N bench.py --gpus $N --steps 3 --warmup 3 --workload qv > gpurun_out/mg${N}_qv.log 2>&1
[ "$N" -ge 4 ] && run $N bench.py --gpus $N --steps 3 --warmup 3 --workload qaoa > gpurun_out/mg${N}_qaoa.log 2>&1
true
