P=30711
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P "${@:2}"; P=$((P+1)); }
run 2 tools/dist_check.py --quick --scale --qft34 > gpurun_out/q2_dc.log 2>&1; echo rc=$? >> gpurun_out/q2_dc.log
run 2 bench.py --gpus 2 --steps 3 --warmup 3 --workload qv > gpurun_out/q2_qv.log 2>&1
run 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/q2_qft.log 2>&1
true
