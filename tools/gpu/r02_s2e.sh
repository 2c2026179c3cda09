set -x
P="16,16,5,k11m10k5m6 24,8,7,k4m8k4m16 27,4,4,k2m6k2m21 23,9,7,k4m3k5m20 23,9,7,k3m1k6m22 26,6,6,k3m1k3m25 24,6,8,k5m4k1m20 22,10,9,k9m14k1m8 22,10,6,k9m15k1m7 23,8,7,k6m17k2m6"
TN_GATHER_DEBUG=1 timeout 300 python tools/gather_bench.py $P 2>&1 | grep -v "^gather" 
for m in 1 2 3; do echo mode $m; TN_GATHER_MODE=$m timeout 300 python tools/gather_bench.py $P 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_chalf -s 1 -c 1 -o gpurun_out/s2e_g31 python tools/gather_bench.py 16,16,5,k11m10k5m6 > gpurun_out/s2e_ncu1.log 2>&1; tail -1 gpurun_out/s2e_ncu1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_chalf -s 1 -c 1 -o gpurun_out/s2e_g4 python tools/gather_bench.py 24,8,7,k4m8k4m16 > gpurun_out/s2e_ncu2.log 2>&1; tail -1 gpurun_out/s2e_ncu2.log
