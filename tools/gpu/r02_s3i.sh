set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/s3i_tests.log 2>&1
tail -5 gpurun_out/s3i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3i_smoke.log 2>&1; tail -4 gpurun_out/s3i_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3i_bench.json 2> gpurun_out/s3i_bench.err; tail -c 400 gpurun_out/s3i_bench.json
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/s3i_ncu_launch.log 2>&1; tail -2 gpurun_out/s3i_ncu_launch.log
gzip -kf gpurun_out/r02b_launches_c3.csv
