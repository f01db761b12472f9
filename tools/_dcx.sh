N=$1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30411 tools/dist_check.py --quick --scale --qft34 > gpurun_out/mgc${N}.log 2>&1; echo rc=$? >> gpurun_out/mgc${N}.log
