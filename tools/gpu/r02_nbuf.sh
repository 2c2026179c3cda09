# tc2 epilogue staging depth A/B (TN_TC2_NBUF 2 vs auto=4 for K <= 2^7), interleaved on one box
for r in 1 2; do
for v in 2 0; do
  TN_TC2_NBUF=$v timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/nbuf_${v}_$r.log 2>&1
  echo "nbuf=$v rep=$r $(tail -1 gpurun_out/nbuf_${v}_$r.log)"
done; done
for v in 2 0; do echo "== $v"; grep -E "^ +(1|3|24|26) m" gpurun_out/nbuf_${v}_2.log; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "tc2 or pair" > gpurun_out/nbuf_tests.log 2>&1; tail -2 gpurun_out/nbuf_tests.log
