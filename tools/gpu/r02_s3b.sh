NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do for v in pack nopack; do
if [ $v = nopack ]; then export TN_NO_PACK=1; else unset TN_NO_PACK; fi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2959$r tools/step_profile_mgpu.py c3 3 > gpurun_out/s3b_sp_${v}_$r.log 2> /dev/null
echo "$v $r: $(tail -n 1 gpurun_out/s3b_sp_${v}_$r.log)"; grep "  5 m25" gpurun_out/s3b_sp_${v}_$r.log
done; done
