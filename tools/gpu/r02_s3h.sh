for r in 1 2; do for v in "TN_PERM_CTAS=2" "TN_PERM_CTAS=3" "TN_PERM_CTAS=4" "TN_PERM_UX=0" "TN_PERM_UX=2"; do
env $v timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3h.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3h.log | cut -c1-120)"
done; done
