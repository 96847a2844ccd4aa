set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python tools/gpu_debug.py > gpurun_out/dbg1.log 2>&1; echo "dbg rc=$?"
tail -5 gpurun_out/dbg1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest1.log
