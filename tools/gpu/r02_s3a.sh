timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -m gpu -q -x > gpurun_out/s3a_t.log 2>&1; tail -3 gpurun_out/s3a_t.log
for v in pack nopack; do
if [ $v = nopack ]; then export TN_NO_PACK=1; else unset TN_NO_PACK; fi
echo $v; timeout 300 python tools/mubench.py --m 27 --k 4 --n 4 --iters 5 2>&1 | tail -1
timeout 300 python tools/gather_bench.py 27,4,4,k2m6k2m21 27,4,4,k4m27 2>&1 | grep -v "^gather"
done
unset TN_NO_PACK
for r in 1 2; do for v in pack nopack; do
if [ $v = nopack ]; then export TN_NO_PACK=1; else unset TN_NO_PACK; fi
timeout 600 python tools/step_profile.py c3 3 20 3 > gpurun_out/s3a_sp_${v}_$r.log 2>&1
echo "$v rep $r: $(tail -n 1 gpurun_out/s3a_sp_${v}_$r.log)"; grep "  5 m27" gpurun_out/s3a_sp_${v}_$r.log
done; done
