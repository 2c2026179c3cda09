for r in 1 2; do for o in 0 1; do
TN_TC2_ORDER=$o timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2m_sp_o${o}_$r.log 2>&1
done; done
for r in 1 2; do for o in 0 1; do echo "order $o rep $r: $(tail -n 1 gpurun_out/s2m_sp_o${o}_$r.log)"; done; done
paste <(cut -c1-90 gpurun_out/s2m_sp_o0_1.log) <(cut -c40-62 gpurun_out/s2m_sp_o1_1.log) <(cut -c40-62 gpurun_out/s2m_sp_o0_2.log) <(cut -c40-62 gpurun_out/s2m_sp_o1_2.log)
