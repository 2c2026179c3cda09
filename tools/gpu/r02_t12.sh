set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_postselect.py tests/test_gpu_loopback.py -m gpu -q --timeout 900 -rf -k "gather or fused or c1_full or c2_reduced or postselect or post_selection or fp16_vs_one" > gpurun_out/t12.log 2>&1
tail -5 gpurun_out/t12.log
python tools/step_profile.py c3 0 20 > gpurun_out/sp2_c3_p0.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_w.json 2> gpurun_out/bench_c3_w.err
python bench.py --plan c5 --steps 3 --warmup 2 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -2 gpurun_out/bench_c5.err
