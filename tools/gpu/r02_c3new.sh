set -x
python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 600 -k "batched or padded" -rA > gpurun_out/t4.log 2>&1
python tools/step_profile.py c3 2 20 > gpurun_out/sp_c3_p2.log 2>&1
python tools/step_profile.py c3 0 20 > gpurun_out/sp_c3_p0.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_p2.json 2> gpurun_out/bench_c3_p2.err
python bench.py --steps 5 --warmup 3 --policy 0 --no-cpu > gpurun_out/bench_c3_p0.json 2> gpurun_out/bench_c3_p0.err
python bench.py --steps 5 --warmup 3 --plan c3_sweep --no-cpu > gpurun_out/bench_c3sweep.json 2> gpurun_out/bench_c3sweep.err
tail -3 gpurun_out/t4.log
