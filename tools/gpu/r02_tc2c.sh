set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "tensor_core_vs_oracle or scaled_gemm" > gpurun_out/tc2d.log 2>&1; tail -2 gpurun_out/tc2d.log
for o in 0 1; do
  TN_TC2_ORDER=$o timeout 600 python tools/mubench.py --m 23 --k 8-10 --n 8-10 --iters 5 > gpurun_out/mb_order$o.txt 2>&1
done
cat gpurun_out/mb_order0.txt gpurun_out/mb_order1.txt
TN_TC2_ORDER=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:tc2 -c 1 python tools/mubench.py --m 23 --k 10 --n 10 --iters 1 > gpurun_out/ncu_order1.log 2>&1
tail -8 gpurun_out/ncu_order1.log
for r in 1 2; do
  for t in 1 0; do
    TN_TC2=$t timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/bench_tc2_${t}_$r.json 2> gpurun_out/bench_tc2_${t}_$r.err
  done
done
python - <<'PY'
import json
for r in (1,2):
    for t in (1,0):
        try:
            d=json.loads([l for l in open(f"gpurun_out/bench_tc2_{t}_{r}.json") if l.startswith("{")][0])
            print(r, "tc2" if t else "tc1", round(d["ms_per_step"],2), "J/step", round(d["energy"]["joules_per_step"],1), "MHz", d["clocks"]["sm_mhz"], d["breakdown_ms"])
        except Exception as e:
            print(r, t, "err", e)
PY
