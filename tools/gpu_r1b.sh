set -x
timeout 300 python tools/gpu_debug.py > gpurun_out/dbg.log 2>&1; echo "dbg rc=$?"
grep -v ": ok" gpurun_out/dbg.log | head -40
grep "uniform20M\|circle1M\|disk2M" gpurun_out/dbg.log
timeout 300 python tools/prof_once.py uniform 2e7 4 > gpurun_out/prof_once.log 2>&1; echo "prof rc=$?"
cat gpurun_out/prof_once.log
