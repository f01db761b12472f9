timeout 1200 python -m pytest tests/test_family_parity.py tests/test_scale_gpu.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/dp_tests.log 2>&1; echo rc=$? >> gpurun_out/dp_tests.log
SVB200_DIAG_PAIRS=0 timeout 600 python tools/qv_sweep_table.py mirror_qaoa31_h29-12 > gpurun_out/dp0.log 2>&1
timeout 600 python tools/qv_sweep_table.py mirror_qaoa31_h29-12 > gpurun_out/dp1.log 2>&1
SVB200_DIAG_PAIRS=0 timeout 600 python tools/qv_sweep_table.py mirror_sup31_h29-12 > gpurun_out/dp0s.log 2>&1
timeout 600 python tools/qv_sweep_table.py mirror_sup31_h29-12 > gpurun_out/dp1s.log 2>&1
