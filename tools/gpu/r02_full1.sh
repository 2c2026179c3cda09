set -x
python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/t9.log 2>&1
timeout 900 python tools/debug_parity.py c3 20 > gpurun_out/dbg5_c3.log 2>&1
tail -15 gpurun_out/t9.log
