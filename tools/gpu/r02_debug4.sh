set -x
python -m pytest tests/test_gpu_sparse_state.py tests/test_gpu_e2e.py -m gpu -q --timeout 900 -k "sparse or recompute or split or c3" -rA > gpurun_out/t8.log 2>&1
timeout 900 python tools/debug_parity.py c3 20,24 > gpurun_out/dbg4_c3.log 2>&1
timeout 600 python tools/debug_parity.py c3_sweep 22 > gpurun_out/dbg4_c3sweep.log 2>&1
python bench.py --steps 5 --warmup 3 --policy 0 > gpurun_out/bench_c3j_p0.json 2> gpurun_out/bench_c3j_p0.err
tail -3 gpurun_out/t8.log
