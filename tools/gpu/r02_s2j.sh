NG=$(nvidia-smi -L | wc -l)
for g in 1 0; do
TN_GRAPH_NCCL=$g timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2954$g bench.py --gpus $NG --steps 8 --warmup 3 --no-cpu > gpurun_out/s2j_bench_n${NG}_g$g.json 2> gpurun_out/s2j_bench_n${NG}_g$g.err
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/s2j_bench_n${NG}_g$g.json") if l.startswith("{")][0])
print("graph_nccl=$g", round(d["ms_per_step"],2), round(d["value"]), d["breakdown_ms"], d["clocks"]["sm_mhz"], d["config"].get("epilogue_swaps"), d["e2e"]["ms_per_step"])
PY
tail -2 gpurun_out/s2j_bench_n${NG}_g$g.err
done
