set -x
python -m pytest tests/test_gpu_e2e.py -m gpu -q --timeout 900 -rf -k "c1_full or c2_reduced or policies" > gpurun_out/t16.log 2>&1
tail -3 gpurun_out/t16.log
python tools/step_profile.py c3 3 20 > gpurun_out/sp5_c3_p3.log 2>&1
python bench.py --steps 5 --warmup 3 --policy 3 --no-cpu > gpurun_out/bench_c3_p3c.json 2> gpurun_out/bench_c3_p3c.err
python bench.py --steps 5 --warmup 3 --policy 0 --no-cpu > gpurun_out/bench_c3_p0c.json 2> gpurun_out/bench_c3_p0c.err
python bench.py --plan c3_sweep --steps 5 --warmup 3 --policy 3 --no-cpu > gpurun_out/bench_c3sw_p3.json 2> gpurun_out/bench_c3sw_p3.err
tail -2 gpurun_out/sp5_c3_p3.log
