TN_GATHER_DEBUG=1 timeout 600 python tools/step_profile.py c3 3 20 1 2> gpurun_out/s3c_modes.err > /dev/null; sort -u gpurun_out/s3c_modes.err | head -20
for r in 1 2; do for v in def raw128; do
if [ $v = raw128 ]; then export TN_RAW_BELOW=128; else unset TN_RAW_BELOW; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3c_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3c_sp_${v}_$r.log)"; grep -E "^  (4|5|8|9|10|13|18|25|26|31) m" gpurun_out/s3c_sp_${v}_$r.log | cut -c1-75
done; done
