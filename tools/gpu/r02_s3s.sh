for t in 1 0; do
TN_TC2=$t timeout 300 python tools/mubench.py --m 25 --k 5-7 --n 6-8 --iters 5 2>&1 | grep -E "^ +[0-9]" | sed "s/^/tc2=$t /"
done
