set -x
timeout 300 python tools/mubench.py --m 27 --k 4 --n 4 --iters 5 2>&1 | tail -1
timeout 300 python tools/mubench.py --m 26 --k 5 --n 6 --iters 5 2>&1 | tail -1
timeout 300 python tools/mubench.py --m 16 --k 16 --n 5 --iters 5 2>&1 | tail -1
timeout 300 python tools/mubench.py --m 21 --k 11 --n 11 --iters 5 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_chalf -s 2 -c 1 -o gpurun_out/s2d_k4n4 python tools/mubench.py --m 27 --k 4 --n 4 --iters 1 > gpurun_out/s2d_ncu1.log 2>&1; tail -2 gpurun_out/s2d_ncu1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_chalf -s 2 -c 1 -o gpurun_out/s2d_m16k16n5 python tools/mubench.py --m 16 --k 16 --n 5 --iters 1 > gpurun_out/s2d_ncu2.log 2>&1; tail -2 gpurun_out/s2d_ncu2.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2 -s 2 -c 1 -o gpurun_out/s2d_tc2_m21k11n11 python tools/mubench.py --m 21 --k 11 --n 11 --iters 1 > gpurun_out/s2d_ncu3.log 2>&1; tail -2 gpurun_out/s2d_ncu3.log
