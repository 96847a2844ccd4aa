# end-of-round evidence (round 2): tests, smoke, bench (+ reference arm), every workload,
# stress vs the compiled reference, sanitizer, ncu launch list + full captures.
# Output: gpurun_out/final/
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --json-out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --l2-flush --no-cpu-baseline --json-out $O/bench_flushed.json > $O/bench_flushed.log 2>&1; echo "bench flushed rc=$?"
timeout 900 python bench.py --impl reference --json-out $O/bench_ref.json > $O/bench_ref.log 2>&1; echo "ref rc=$?"
for w in uniform1m disk20m circle4m; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --json-out $O/bench_$w.json > $O/bench_$w.log 2>&1; echo "$w rc=$?"; done
timeout 600 python bench.py --workload uniform1b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --json-out $O/bench_1b.json > $O/bench_1b.log 2>&1; echo "1b rc=$?"
timeout 1200 python tools/stress.py 400 7 > $O/stress.log 2>&1; echo "stress rc=$?"; tail -1 $O/stress.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 $O/memcheck.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_once.py uniform 2e7 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_classify|k3_round1|k_rounds" -c 4 -o $O/prof_uniform python tools/prof_once.py uniform 2e7 1 > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rounds" -c 1 -o $O/prof_disk_kr python tools/prof_once.py disk 2e7 1 > /dev/null 2>&1; echo "ncu3 rc=$?"
SHB_LIB=build_var/lib_probes.so TRACE_ROUND=255 python tools/prof_once.py uniform 2e7 3 > $O/probe_uniform.txt 2>&1  # probes build: tools/build_var.sh probes -DSHB_PROBES
python tools/prof_once.py disk 2e7 2 > $O/phases_disk.txt 2>&1
python tools/prof_once.py circle 4e6 2 > $O/phases_circle.txt 2>&1
