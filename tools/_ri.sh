timeout 900 python -m pytest tests/test_family_parity.py tests/test_scale_gpu.py -m gpu -q -x > gpurun_out/ri_tests.log 2>&1; echo rc=$? >> gpurun_out/ri_tests.log
SVB200_JIT_REAL_IMAG_FMA=0 timeout 600 python tools/qv_sweep_table.py mirror_qaoa31_h29-12 > gpurun_out/ri0.log 2>&1
timeout 600 python tools/qv_sweep_table.py mirror_qaoa31_h29-12 > gpurun_out/ri1.log 2>&1
SVB200_JIT_REAL_IMAG_FMA=0 timeout 600 python tools/qv_sweep_table.py mirror_sup31_h29-12 > gpurun_out/ri0s.log 2>&1
timeout 600 python tools/qv_sweep_table.py mirror_sup31_h29-12 > gpurun_out/ri1s.log 2>&1
