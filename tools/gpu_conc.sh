# two processes on one GPU: merge-hull determinism per library variant / payload width
for v in build_var/lib_cur.so build_var/lib_prelf.so; do
  for w in 512 2048; do
    echo "== $v width $w"
    (SHB_LIB=$v python tools/dbg_merge2.py 100 $w & SHB_LIB=$v python tools/dbg_merge2.py 100 $w & wait)
  done
done
