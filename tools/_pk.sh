P=30611
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P "${@:2}"; P=$((P+1)); }
run 4 tools/dist_check.py --quick --scale > gpurun_out/pk_dc.log 2>&1; echo rc=$? >> gpurun_out/pk_dc.log
run 4 bench.py --gpus 4 --steps 3 --warmup 3 --workload qaoa > gpurun_out/pk_qaoa.log 2>&1
run 4 bench.py --gpus 4 --steps 3 --warmup 3 --workload qv > gpurun_out/pk_qv.log 2>&1
true
