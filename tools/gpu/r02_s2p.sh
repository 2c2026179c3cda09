timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "mn_ or gathered_runs or tensor_core or scaled" > gpurun_out/s2p_k.log 2>&1; tail -3 gpurun_out/s2p_k.log
for s in "22 9 8 11" "21 10 8 10" "21 11 11 11" "22 10 9 11"; do timeout 300 python tools/mn_bench.py $s 5; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2 -s 1 -c 1 -o gpurun_out/s2p_mn python tools/mn_bench.py 22 9 8 11 1 > gpurun_out/s2p_ncu.log 2>&1; tail -1 gpurun_out/s2p_ncu.log
