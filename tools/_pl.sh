for cfg in "SVB200_BENCH_PIPELINE=0" "" "SVB200_BENCH_PIPELINE=0" ""; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --sub-steps 0 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['roofline']['per_sweep_ms'], d['config']['circuits_in_flight'])" >> gpurun_out/pl.log
done
timeout 900 python bench.py > gpurun_out/pl_full.log 2>&1
