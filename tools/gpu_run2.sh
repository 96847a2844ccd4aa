set -x
python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench_uniform20m.json > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench2.log
for w in disk20m circle4m; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_$w.json >> gpurun_out/bench2.log 2>&1; done
python tools/prof_once.py uniform 2e7 3 > gpurun_out/prof_once.log 2>&1
python tools/prof_once.py disk 2e7 3 >> gpurun_out/prof_once.log 2>&1
python tools/prof_once.py circle 4e6 3 >> gpurun_out/prof_once.log 2>&1
cat gpurun_out/prof_once.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_uniform20m.csv python tools/prof_once.py uniform 2e7 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_classify|k3_route|k4_table" -c 8 -o gpurun_out/prof_uniform20m python tools/prof_once.py uniform 2e7 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -5 gpurun_out/ncu_full.log
