timeout 900 python -m pytest tests/test_broadcast_merge.py tests/test_scale_gpu.py tests/test_family_parity.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/bm_tests.log 2>&1; echo rc=$? >> gpurun_out/bm_tests.log
rm -f gpurun_out/bm.log
for cfg in "SVB200_BROADCAST_MERGE=0" "" "SVB200_BROADCAST_MERGE=0" ""; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --sub-steps 0 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['roofline']['per_sweep_ms'], d['roofline']['frac'], d['roofline']['kernel'])" >> gpurun_out/bm.log
done
