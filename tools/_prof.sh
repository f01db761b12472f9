timeout 600 python tools/prof_sweep.py qft30_h30-12 > gpurun_out/prof_pre.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svb_jit_ --launch-skip 2 --launch-count 1 -o gpurun_out/qft30_bcast -f python tools/prof_sweep.py qft30_h30-12 > gpurun_out/prof_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bcast.csv python bench.py --steps 2 --warmup 3 --sub-steps 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof_launch.log 2>&1
echo done >> gpurun_out/prof_full.log
