cp paper_2407_00769_b200/libtn.so /tmp/libtn_nb2.so
for r in 1 2; do for v in 2 4; do
cp /tmp/libtn_nb2.so paper_2407_00769_b200/libtn.so; if [ $v = 4 ]; then cp paper_2407_00769_b200/libtn_nb4.so paper_2407_00769_b200/libtn.so; fi
touch paper_2407_00769_b200/libtn.so
timeout 300 python tools/mubench.py --m 20 --k 4-6 --n 10-12 --iters 5 2>&1 | grep -E "^ +[0-9]" | awk -v v=$v '{print "nbuf="v, $1, $2, $3, $7}'
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s4d_sp.log 2>&1
echo "nbuf=$v rep $r: $(tail -n 1 gpurun_out/s4d_sp.log)"; grep -E " (3|9|12|17|20|24) m" gpurun_out/s4d_sp.log | cut -c1-75
done; done
cp /tmp/libtn_nb2.so paper_2407_00769_b200/libtn.so
