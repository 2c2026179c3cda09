# interleaved A/B: tc1 epilogue fast path (repo) vs previous build (ab_old/, git-ignored copy)
for r in 1 2 3; do
  timeout 300 python tools/step_profile.py c3 3 20 3 > gpurun_out/ab_new_$r.log 2>&1
  (cd ab_old && timeout 300 python tools/step_profile.py c3 3 20 3 > ../gpurun_out/ab_old_$r.log 2>&1)
  for v in new old; do
    echo "$v r=$r $(tail -1 gpurun_out/ab_${v}_$r.log | cut -c1-150)"
    grep -E "^ +(3|13|14|28|29) m" gpurun_out/ab_${v}_$r.log | awk '{printf "%s:%s ", $1, $12} END {print ""}'
  done
done
