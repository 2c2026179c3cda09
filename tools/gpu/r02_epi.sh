# tc1 epilogue without per-value selects on full chunks: parity tests, mubench, step profile
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -x -q > gpurun_out/epi_tests.log 2>&1; tail -1 gpurun_out/epi_tests.log
timeout 300 python tools/mubench.py --m 26 --k 5 --n 6 --iters 5 > gpurun_out/epi_mub.log 2>&1; tail -1 gpurun_out/epi_mub.log
timeout 300 python tools/mubench.py --m 27 --k 4 --n 4 --iters 5 >> gpurun_out/epi_mub.log 2>&1; tail -1 gpurun_out/epi_mub.log
for r in 1 2; do
  timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/epi_sp_$r.log 2>&1
  tail -1 gpurun_out/epi_sp_$r.log | cut -c1-170
  grep -E "^ +(13|14|28|29|30) m" gpurun_out/epi_sp_$r.log | awk '{printf "%s:%s ", $1, $12} END {print ""}'
done
