NG=$(nvidia-smi -L | wc -l)
if [ $NG = 1 ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s2w_bench_n1.json 2> gpurun_out/s2w_bench_n1.err
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s2w_bench_n1b.json 2> gpurun_out/s2w_bench_n1b.err
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2w_ref_n1.json 2> gpurun_out/s2w_ref_n1.err
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $NG --steps 8 --warmup 3 > gpurun_out/s2w_bench_n$NG.json 2> gpurun_out/s2w_bench_n$NG.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus $NG --steps 8 --warmup 3 > gpurun_out/s2w_bench_n${NG}b.json 2> gpurun_out/s2w_bench_n${NG}b.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus $NG --steps 5 --warmup 3 --replicas > gpurun_out/s2w_bench_n${NG}_rep.json 2> gpurun_out/s2w_bench_n${NG}_rep.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29564 tools/step_profile_mgpu.py c3 3 > gpurun_out/s2w_sp_n$NG.log 2> /dev/null
fi
for f in gpurun_out/s2w_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
    print(sys.argv[1], d.get("impl", "ours"), round(d.get("ms_per_step", 0), 1), round(d.get("value", 0), 1), d.get("clocks", {}).get("sm_mhz"), d.get("config", {}).get("epilogue_swaps"), d.get("breakdown_ms"))
except Exception as e:
    print(sys.argv[1], "err", e)
PY
done
