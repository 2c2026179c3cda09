timeout 300 python tools/mubench.py --m 27 --k 4 --n 4 --iters 5 2>&1 | tail -1
timeout 300 python tools/mubench.py --m 26 --k 5 --n 6 --iters 5 2>&1 | tail -1
timeout 300 python tools/mubench.py --m 25 --k 6 --n 4 --iters 5 2>&1 | tail -1
for m in 0 1 2 3; do echo "mode $m"; TN_GATHER_MODE=$m timeout 300 python tools/gather_bench.py 27,4,4,k4m27 26,5,6,k5m26 24,8,7,k4m8k4m16 27,4,4,k2m6k2m21 2>&1 | grep -v "^gather"; done
