for v in build_var/*.so; do echo "== $v"; SHB_LIB=$v timeout 120 python tools/prof_once.py uniform 2e7 3 2>&1 | tail -1; done
echo "== default"; timeout 120 python tools/prof_once.py uniform 2e7 3 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k3_round1" -c 2 -o gpurun_out/prof_v3 python tools/prof_once.py uniform 2e7 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
