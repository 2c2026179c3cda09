timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "mn_" > gpurun_out/s2q_k.log 2>&1; tail -1 gpurun_out/s2q_k.log
for s in "22 9 8 11" "21 10 8 10" "21 11 11 11" "22 10 9 11"; do timeout 300 python tools/mn_bench.py $s 5; done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc2 -c 2 python tools/mn_bench.py 22 9 8 11 1 2>&1 | grep -E "tc2_kernel|duration|tensor|conflicts|wavefronts|per_second" | head -14
for r in 1 2; do for m in 0 1; do
if [ $m = 1 ]; then export TN_NO_MN=1; else unset TN_NO_MN; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s2q_sp_nomn${m}_$r.log 2>&1
echo "nomn=$m rep $r: $(tail -n 1 gpurun_out/s2q_sp_nomn${m}_$r.log)"
done; done
