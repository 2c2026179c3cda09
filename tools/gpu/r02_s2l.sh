for o in 0 1; do
  TN_TC2_ORDER=$o timeout 300 python tools/mubench.py --m 21 --k 10-11 --n 10-11 --iters 5 2>&1 | grep -E "^ +1[01] +1[01]" | sed "s/^/order $o /"
  TN_TC2_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc2 -c 8 --csv python tools/mubench.py --m 21 --k 10-11 --n 10-11 --iters 1 2>/dev/null | grep -E "tc2" | awk -F'","' '{print "order '$o'", $5, $(NF-2), $(NF-1), $NF}' | sed 's/"//g' | head -24
done
