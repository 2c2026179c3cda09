# output-heavy tc2 shape (C3 step 3: m20 k6 n12, identity output): time, then one ncu --set full capture
timeout 300 python tools/mubench.py --m 20 --k 6 --n 12 --iters 5 > gpurun_out/oh_mub.log 2>&1; tail -3 gpurun_out/oh_mub.log
timeout 300 python tools/mubench.py --m 23 --k 6 --n 9 --iters 5 >> gpurun_out/oh_mub.log 2>&1; tail -2 gpurun_out/oh_mub.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_chalf -s 2 -c 1 -o gpurun_out/r02_gemm_tc2_m20k6n12 -f python tools/mubench.py --m 20 --k 6 --n 12 --iters 1 > gpurun_out/oh_ncu.log 2>&1; tail -2 gpurun_out/oh_ncu.log
