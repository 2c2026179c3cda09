# permutation-pass tuning knobs on the C3 subtask, interleaved (perm total per subtask)
for r in 1 2 3; do
  for v in "X=0" "TN_PERM_CTAS=3" "TN_PERM_CTAS=1" "TN_PERM_UX=0"; do
    env $v timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/pa.log 2>&1
    echo "$v r=$r $(tail -1 gpurun_out/pa.log | grep -o "perm [0-9.]*") $(tail -1 gpurun_out/pa.log | grep -o 'sum median [0-9.]*')"
  done
done
