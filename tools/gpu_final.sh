# end-of-round evidence: tests, smoke, bench (+ reference arm), workloads, ncu launch list + full capture
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --json-out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --json-out gpurun_out/bench_ref.json > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
for w in disk20m circle4m; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"; done
timeout 600 python bench.py --workload uniform1b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_1b.json > gpurun_out/bench_1b.log 2>&1; echo "1b rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/prof_once.py uniform 2e7 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_classify|k3_round1|k_rounds" -c 4 -o gpurun_out/prof_final python tools/prof_once.py uniform 2e7 1 > /dev/null 2>&1; echo "ncu2 rc=$?"
