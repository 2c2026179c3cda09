NG=$(nvidia-smi -L | wc -l)
TN_DEBUG_COMPOSE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29671 tools/step_profile_mgpu.py c3 3 > gpurun_out/comp2_sp.log 2> gpurun_out/comp2_sp.err
grep -m4 "compose" gpurun_out/comp2_sp.err
grep " 14 m" gpurun_out/comp2_sp.log
TN_NO_SWAP_COMPOSE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29672 tools/step_profile_mgpu.py c3 3 > gpurun_out/comp2_sp1.log 2>/dev/null
grep " 14 m\|sum" gpurun_out/comp2_sp1.log
