timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v_tests.log 2>&1; echo rc=$? >> gpurun_out/v_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo rc=$? >> gpurun_out/v_smoke.log
timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1
