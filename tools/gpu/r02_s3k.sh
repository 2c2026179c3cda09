for h in 1 0; do
TN_L2_HINTS=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc2 -s 1 -c 1 python tools/mubench.py --m 21 --k 11 --n 11 --iters 1 2>&1 | grep -E "duration|dram__bytes|hit_rate|per_second" | sed "s/^/hints=$h /"
TN_L2_HINTS=$h timeout 300 python tools/mubench.py --m 21 --k 9-11 --n 10-11 --iters 5 2>&1 | grep -E "^ +(9|10|11) " | sed "s/^/hints=$h /"
done
for r in 1 2; do for h in 1 0; do
TN_L2_HINTS=$h timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3k_sp_$h.log 2>&1
echo "hints=$h rep $r: $(tail -n 1 gpurun_out/s3k_sp_$h.log | cut -c1-130)"; grep " 30 m21" gpurun_out/s3k_sp_$h.log | cut -c1-90
done; done
