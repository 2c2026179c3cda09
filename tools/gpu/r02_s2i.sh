NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29531 tools/step_profile_mgpu.py c3 3 > gpurun_out/s2i_sp_n$NG.log 2> gpurun_out/s2i_sp_n$NG.err
cat gpurun_out/s2i_sp_n$NG.log; tail -3 gpurun_out/s2i_sp_n$NG.err
