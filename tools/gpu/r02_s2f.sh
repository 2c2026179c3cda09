set -x
nvidia-smi -L
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/s2f_n4.json 2> gpurun_out/s2f_n4.err; tail -c 2500 gpurun_out/s2f_n4.json; tail -5 gpurun_out/s2f_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/s2f_n2.json 2> gpurun_out/s2f_n2.err; tail -c 2500 gpurun_out/s2f_n2.json; tail -5 gpurun_out/s2f_n2.err
