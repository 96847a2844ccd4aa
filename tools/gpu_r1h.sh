timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --workload uniform1b --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_1b.json > gpurun_out/bench_1b.log 2>&1; echo "1b rc=$?"; tail -2 gpurun_out/bench_1b.log
python tools/prof_once.py circle 4e6 2 > gpurun_out/prof_circle.log 2>&1
python tools/prof_once.py disk 2e7 2 > gpurun_out/prof_disk.log 2>&1
