set -x
python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/t17.log 2>&1
tail -8 gpurun_out/t17.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final1.json 2> gpurun_out/bench_final1.err
python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_run2.log 2>&1
tail -2 gpurun_out/ncu_run2.log
