for r in 1 2 3; do for m in 28 32 99; do
TN_MN_MIN_LOG2=$m timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2r_sp_mn${m}_$r.log 2>&1
echo "mn_min=$m rep $r: $(tail -n 1 gpurun_out/s2r_sp_mn${m}_$r.log)"
done; done
paste <(cut -c1-62 gpurun_out/s2r_sp_mn32_1.log) <(cut -c28-62 gpurun_out/s2r_sp_mn99_1.log) | tail -6
