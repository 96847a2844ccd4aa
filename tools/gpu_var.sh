# round phases of circle 4M for every library variant in build_var/
for v in build_var/*.so; do echo "== $v"; SHB_LIB=$v timeout 120 python tools/prof_once.py circle 4e6 2 > /tmp/o.log 2>&1; echo rc=$?; tail -30 /tmp/o.log | grep -E "round (1[0-9]|2[0-9])|KernelTim|Error|error|CTA" | sed 's/KernelTimings.*PhaseTimings/ /'; tail -3 /tmp/o.log; done
for t in 12 20; do echo "== trace $t"; TRACE_ROUND=$t timeout 120 python tools/prof_once.py circle 4e6 1 2>&1 | grep -E "CTA|round $t:"; done
