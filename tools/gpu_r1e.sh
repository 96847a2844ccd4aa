timeout 300 python tools/gpu_debug.py > gpurun_out/dbg.log 2>&1; echo "dbg rc=$?"; grep -v ": ok" gpurun_out/dbg.log | head; grep -c ": ok" gpurun_out/dbg.log
timeout 300 python tools/prof_once.py uniform 2e7 4 > gpurun_out/prof_once.log 2>&1; tail -2 gpurun_out/prof_once.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_classify|k3_round1|k_rounds" -c 4 -o gpurun_out/prof_v4 python tools/prof_once.py uniform 2e7 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
