# 4 GPUs: per-step cost of epilogue swaps vs peer-pass swaps (TN_NO_EPILOGUE_SWAP=1), interleaved
NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do
for v in 0 1; do
  TN_NO_EPILOGUE_SWAP=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 298$r$v tools/step_profile_mgpu.py c3 3 > gpurun_out/ss_${v}_$r.log 2>/dev/null
  echo "noepi=$v r=$r $(tail -1 gpurun_out/ss_${v}_$r.log)"
done; done
