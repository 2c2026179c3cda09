# gather-vs-pass time model A/B (TN_GATHER_ALWAYS=1 = gather whenever the layout allows), interleaved
NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do
for v in 1 0; do
  TN_GATHER_ALWAYS=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 297$r$v bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/gm_n${NG}_${v}_$r.json 2> gpurun_out/gm_n${NG}_${v}_$r.err
  python - gpurun_out/gm_n${NG}_${v}_$r.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][0])
print(sys.argv[1], round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], {k: round(v, 2) for k, v in d["breakdown_ms"].items()})
PY
done; done
