set -x
export NCCL_DEBUG=WARN
python -m pytest tests/test_gpu_multi.py -m gpu -q --timeout 1500 -rf -s > gpurun_out/multi_t.log 2>&1
tail -5 gpurun_out/multi_t.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
$TR --nproc-per-node 2 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
$TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
$TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --steps 5 --warmup 3 --quant-from-pct 0 > gpurun_out/bench_n4_int8all.json 2> gpurun_out/bench_n4_int8all.err
$TR --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --steps 5 --warmup 3 --comm fp16 > gpurun_out/bench_n4_fp16.json 2> gpurun_out/bench_n4_fp16.err
$TR --nproc-per-node 4 --master-port 29615 bench.py --gpus 4 --steps 5 --warmup 3 --replicas > gpurun_out/bench_n4_rep.json 2> gpurun_out/bench_n4_rep.err
$TR --nproc-per-node 4 --master-port 29616 bench.py --gpus 4 --steps 3 --warmup 2 --plan c5 > gpurun_out/bench_n4_c5.json 2> gpurun_out/bench_n4_c5.err
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_n1_same.json 2> gpurun_out/bench_n1_same.err
tail -3 gpurun_out/bench_n4.err
