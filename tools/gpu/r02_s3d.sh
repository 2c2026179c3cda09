for r in 1 2 3; do for v in def praw; do
if [ $v = praw ]; then export TN_PLAIN_RAW=1; else unset TN_PLAIN_RAW; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3d_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3d_sp_${v}_$r.log)"; grep -E " (28|29|9|4) m" gpurun_out/s3d_sp_${v}_$r.log | cut -c1-75
done; done
