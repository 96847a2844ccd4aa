# large-table path: parity sweep + circle/disk round phases
timeout 400 python tools/gpu_debug.py > gpurun_out/dbg.log 2>&1; echo "dbg rc=$?"; grep -v ": ok" gpurun_out/dbg.log | head -20; grep -c ": ok" gpurun_out/dbg.log
timeout 200 python tools/prof_once.py circle 4e6 2 > gpurun_out/circ.log 2>&1; echo "circ rc=$?"
timeout 200 python tools/prof_once.py disk 2e7 2 > gpurun_out/disk.log 2>&1; echo "disk rc=$?"
grep KernelTimings gpurun_out/circ.log gpurun_out/disk.log | sed 's/KernelTimings.*PhaseTimings/ /'
