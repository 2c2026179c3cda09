set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/s2n_tests.log 2>&1
tail -6 gpurun_out/s2n_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2n_smoke.log 2>&1; tail -4 gpurun_out/s2n_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s2n_bench.json 2> gpurun_out/s2n_bench.err; tail -c 1500 gpurun_out/s2n_bench.json
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/s2n_ncu_launch.log 2>&1; tail -3 gpurun_out/s2n_ncu_launch.log
gzip -kf gpurun_out/r02_launches_c3.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2 -s 2 -c 1 -o gpurun_out/r02_gemm_tc2_m21k11n11 python tools/mubench.py --m 21 --k 11 --n 11 --iters 1 > gpurun_out/s2n_ncu_full.log 2>&1; tail -2 gpurun_out/s2n_ncu_full.log
