rm -f gpurun_out/rb.log
for cfg in "" "SVB200_JIT_RB=3" "" "SVB200_JIT_RB=3"; do
  env $cfg timeout 900 python bench.py --steps 20 --warmup 5 --sub-steps 6 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); q=d['sub']['qv30_h30-12']; print('$cfg', d['ms_per_step'], d['roofline']['per_sweep_ms'], q['circuit_ms'], q['dominant']['launch_ms'], q['fp64_all_sweeps']['frac'])" >> gpurun_out/rb.log
done
