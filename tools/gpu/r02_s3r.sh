for t in 1 0; do
TN_TC2=$t timeout 300 python tools/mubench.py --m 24 --k 8 --n 7 --iters 5 2>&1 | tail -1 | sed "s/^/tc2=$t m24 /"
TN_TC2=$t timeout 300 python tools/mubench.py --m 26 --k 6 --n 6 --iters 5 2>&1 | tail -1 | sed "s/^/tc2=$t m26 /"
TN_TC2=$t timeout 300 python tools/mubench.py --m 23 --k 9 --n 7 --iters 5 2>&1 | tail -1 | sed "s/^/tc2=$t m23 /"
done
for m in 3 2; do TN_GATHER_MODE=$m timeout 300 python tools/gather_bench.py 24,8,7,k4m8k4m16 26,6,6,k3m1k3m25 23,9,7,k3m1k6m22 2>&1 | sed "s/^/mode=$m /"; done
