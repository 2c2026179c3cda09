# output-heavy single-CTA shape (C3 step 29: m26 k5 n6): time + ncu --set full
timeout 300 python tools/mubench.py --m 26 --k 5 --n 6 --iters 5 > gpurun_out/oh2_mub.log 2>&1; tail -2 gpurun_out/oh2_mub.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_chalf -s 2 -c 1 -o gpurun_out/r02_gemm_tc1_m26k5n6 -f python tools/mubench.py --m 26 --k 5 --n 6 --iters 1 > gpurun_out/oh2_ncu.log 2>&1; tail -1 gpurun_out/oh2_ncu.log
