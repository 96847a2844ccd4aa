timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_v2.csv python tools/prof_once.py uniform 2e7 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_classify|k3_round1|k_rounds" -c 4 -o gpurun_out/prof_v2 python tools/prof_once.py uniform 2e7 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_full.log
