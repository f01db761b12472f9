P=29711
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/dist_check.py --quick --scale --qft34 > gpurun_out/mgc2.log 2>&1; echo rc=$? >> gpurun_out/mgc2.log
