set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs -x > gpurun_out/s2s_tests.log 2>&1
tail -6 gpurun_out/s2s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2s_smoke.log 2>&1; tail -4 gpurun_out/s2s_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s2s_bench.json 2> gpurun_out/s2s_bench.err; tail -c 600 gpurun_out/s2s_bench.json
