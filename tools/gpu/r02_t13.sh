set -x
python -m pytest tests/test_gpu_e2e.py tests/test_gpu_kernels.py -m gpu -q --timeout 900 -rf -k "c1_full or c2_reduced or policies or word_pieces" > gpurun_out/t13.log 2>&1
tail -5 gpurun_out/t13.log
python tools/step_profile.py c3 3 20 > gpurun_out/sp3_c3_p3.log 2>&1
python bench.py --steps 5 --warmup 3 --policy 3 --no-cpu > gpurun_out/bench_c3_p3.json 2> gpurun_out/bench_c3_p3.err
python bench.py --steps 5 --warmup 3 --policy 0 --no-cpu > gpurun_out/bench_c3_p0b.json 2> gpurun_out/bench_c3_p0b.err
tail -2 gpurun_out/sp3_c3_p3.log
