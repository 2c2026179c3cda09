# split-block MN-major operand: parity (e2e vs oracle), then interleaved A/B TN_MN_SPLIT=1/0 on the C3 subtask
timeout 1200 python -m pytest tests/test_gpu_e2e.py -x -q -k "mn_major" > gpurun_out/mns_tests.log 2>&1; tail -1 gpurun_out/mns_tests.log
for r in 1 2 3; do
for v in 1 0; do
  TN_MN_SPLIT=$v timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/mns_${v}_$r.log 2>&1
  echo "split=$v r=$r $(tail -1 gpurun_out/mns_${v}_$r.log | cut -c1-160)"
done; done
