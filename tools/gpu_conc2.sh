for cfg in "plain 1024" "ids 1024" "plain 4096" "ids 4096" "ids 50000" "plain 50000"; do
  set -- $cfg
  (python tools/dbg_conc.py $1 $2 200 & python tools/dbg_conc.py $1 $2 200 & wait)
done
