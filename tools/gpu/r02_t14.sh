set -x
TN_STAGE_DEEP=1 python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 600 -k "gemm" > gpurun_out/t14a.log 2>&1
TN_STAGE_DEEP=0 python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 600 -k "gemm" > gpurun_out/t14b.log 2>&1
tail -2 gpurun_out/t14a.log gpurun_out/t14b.log
for r in 1 2; do
TN_STAGE_DEEP=0 python tools/mubench.py --k 6-10 --n 6-10 --out gpurun_out/mb_shallow_$r.txt > /dev/null 2>&1
TN_STAGE_DEEP=1 python tools/mubench.py --k 6-10 --n 6-10 --out gpurun_out/mb_deep_$r.txt > /dev/null 2>&1
done
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_r2a.json 2> gpurun_out/bench_c3_r2a.err
python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_run.log 2>&1
tail -3 gpurun_out/ncu_run.log
