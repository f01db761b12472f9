rm -f gpurun_out/bo.log
for cfg in "" "SVB200_JIT_BCAST_F_OUTER=1" "SVB200_JIT_DIRECT_STORE=0" "" "SVB200_JIT_BCAST_F_OUTER=1" "SVB200_JIT_DIRECT_STORE=0"; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --sub-steps 0 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['roofline']['per_sweep_ms'])" >> gpurun_out/bo.log
done
