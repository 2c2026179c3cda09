# end-of-round launch list of the headline bench (cold, serialised; shares only)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3_end.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/le_ncu.log 2>&1; tail -2 gpurun_out/le_ncu.log
python tools/ncu_summary.py gpurun_out/r02_launches_c3_end.csv 5 gpurun_out/r02_launches_summary_end.json | tail -8
