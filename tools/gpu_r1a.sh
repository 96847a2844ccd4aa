set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep 'Model name'
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest.log
timeout 300 python tools/prof_once.py uniform 2e7 4 > gpurun_out/prof_once.log 2>&1
timeout 300 python tools/prof_once.py uniform 1e6 4 >> gpurun_out/prof_once.log 2>&1
cat gpurun_out/prof_once.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_uniform20m.csv python tools/prof_once.py uniform 2e7 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_classify" -c 1 -o gpurun_out/prof_k2 python tools/prof_once.py uniform 2e7 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --json-out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench.log
