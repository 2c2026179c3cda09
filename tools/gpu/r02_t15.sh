set -x
TN_STAGE_DEEP=1 python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 600 -k "gemm" > gpurun_out/t15a.log 2>&1
python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/t15.log 2>&1
tail -3 gpurun_out/t15a.log; tail -12 gpurun_out/t15.log
TN_STAGE_DEEP=1 python tools/mubench.py --k 8-10 --n 6-10 --out gpurun_out/mb_deep_3.txt > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_r2b.json 2> gpurun_out/bench_c3_r2b.err
python tools/step_profile.py c3 3 20 > gpurun_out/sp4_c3_p3.log 2>&1
python bench.py --steps 5 --warmup 3 --policy 3 --no-cpu > gpurun_out/bench_c3_p3b.json 2> gpurun_out/bench_c3_p3b.err
python bench.py --plan c5 --steps 3 --warmup 2 > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
python bench.py --plan c3_sweep --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3sw_b.json 2> gpurun_out/bench_c3sw_b.err
