#timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ds_tests.log 2>&1; echo rc=$? >> gpurun_out/ds_tests.log
rm -f gpurun_out/ds.log
for cfg in "SVB200_JIT_DIRECT_STORE=0" "" "SVB200_JIT_DIRECT_STORE=0" ""; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --sub-steps 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['roofline']['per_sweep_ms'], d['sub']['qv30_h30-12']['circuit_ms'])" >> gpurun_out/ds.log
done
