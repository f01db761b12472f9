timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:svb_jit_ --launch-skip 2 --launch-count 1 -o gpurun_out/qft30_final_bcast -f python tools/prof_sweep.py qft30_h30-12 > gpurun_out/f_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --sub-steps 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_ncu2.log 2>&1
echo done >> gpurun_out/f_ncu.log
