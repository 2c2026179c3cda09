# swap pass composed with the next step's permutation: tests + interleaved A/B on 2 GPUs
set -x
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "fused_swap" -s > gpurun_out/comp_loop.log 2>&1; tail -5 gpurun_out/comp_loop.log
grep "composed=" gpurun_out/comp_loop.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/comp_multi.log 2>&1; tail -3 gpurun_out/comp_multi.log
for r in 1 2; do
for v in 0 1; do
  TN_NO_SWAP_COMPOSE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2966$r$v bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/comp_n${NG}_${v}_$r.json 2> gpurun_out/comp_n${NG}_${v}_$r.err
  python - gpurun_out/comp_n${NG}_${v}_$r.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print(sys.argv[1], round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], d["breakdown_ms"])
PY
done; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29671 tools/step_profile_mgpu.py c3 3 > gpurun_out/comp_sp_n$NG.log 2>/dev/null
grep -n "pre\|totals" gpurun_out/comp_sp_n$NG.log | sort -t' ' -k7 -rn | head -8
