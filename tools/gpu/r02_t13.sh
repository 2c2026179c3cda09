set -x
python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/t13.log 2>&1
tail -12 gpurun_out/t13.log
python tools/step_profile.py c3 3 20 > gpurun_out/sp3_c3_p3.log 2>&1
python bench.py --steps 5 --warmup 3 --policy 3 --no-cpu > gpurun_out/bench_c3_p3.json 2> gpurun_out/bench_c3_p3.err
python bench.py --steps 5 --warmup 3 --policy 0 --no-cpu > gpurun_out/bench_c3_p0b.json 2> gpurun_out/bench_c3_p0b.err
python tools/mubench.py --k 6-10 --n 6-10 --out gpurun_out/r02_mubench_b.txt > gpurun_out/mubench_b.log 2>&1
tail -2 gpurun_out/sp3_c3_p3.log
