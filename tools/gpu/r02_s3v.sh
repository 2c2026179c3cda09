for r in 1 2 3; do for v in "6,22" "6,30" "30" "none"; do
if [ "$v" = none ]; then E="TN_NO_MN=1"; else E="TN_MN_STEPS=$v"; fi
env $E timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3v_sp.log 2>&1
echo "mn=$v rep $r: $(tail -n 1 gpurun_out/s3v_sp.log | cut -c1-150)"
done; done
