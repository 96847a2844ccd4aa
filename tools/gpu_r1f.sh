timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
for w in disk20m circle4m; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_$w.json >> gpurun_out/bench.log 2>&1; echo "$w rc=$?"; done
python tools/prof_once.py disk 2e7 2 > gpurun_out/prof_disk.log 2>&1; tail -2 gpurun_out/prof_disk.log
