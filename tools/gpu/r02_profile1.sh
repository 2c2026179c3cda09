set -x
python -m pytest tests/test_gpu_loopback.py -m gpu -q --timeout 900 -k "sparse or int8_tensor" -rA > gpurun_out/t3.log 2>&1
python tools/mubench.py --out gpurun_out/r02_mubench.txt > gpurun_out/mubench.log 2>&1
for s in "9 9" "10 10" "10 6" "4 10"; do set -- $s
  python tools/mubench.py --k $1 --n $2 --iters 1 > gpurun_out/mb_$1_$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gemm_chalf -s 2 -c 1 -o gpurun_out/r02_gemm_k$1n$2 python tools/mubench.py --k $1 --n $2 --iters 1 > gpurun_out/ncu_$1_$2.log 2>&1
done
python tools/step_profile.py c3 0 20 > gpurun_out/step_profile.log 2>&1
tail -3 gpurun_out/t3.log
