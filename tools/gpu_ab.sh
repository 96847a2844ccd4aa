# A/B of the library variants in build_var/ on one box: uniform 20M, disk 20M, circle 4M (twice each)
for rep in 1 2; do
python tools/compare_libs.py build_var/*.so
KIND=disk python tools/compare_libs.py build_var/*.so
KIND=circle N=4e6 python tools/compare_libs.py build_var/*.so
done
