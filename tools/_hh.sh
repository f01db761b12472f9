P=29811
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P "${@:2}"; P=$((P+1)); }
run 2 tools/dist_check.py --quick --scale > gpurun_out/hh_dc.log 2>&1; echo rc=$? >> gpurun_out/hh_dc.log
rm -f gpurun_out/hh.log
for cfg in "SVB200_HOST_HANDSHAKE=0" "" ; do
  for wl in qft qv; do
    st=20; [ $wl = qv ] && st=3
    env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps $st --warmup 3 --workload $wl 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$wl', d['ms_per_step'], d['roofline']['all_sweeps']['sweep_ms_per_step'], d.get('e2e') and d['e2e']['ms_per_step'])" >> gpurun_out/hh.log
    P=$((P+1))
  done
done
