# build_var.sh NAME "-DFLAG ..." [SRCROOT]: a variant of the library into build_var/lib_NAME.so
# (SRCROOT: another checkout, e.g. `git worktree add /tmp/head HEAD`, for a same-box A/B)
ROOT=${3:-.}
mkdir -p build_var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -regUsageLevel=8 -Xcompiler -fPIC,-ffp-contract=off,-fopenmp -lgomp -I $ROOT/include -shared $2 -o build_var/lib_$1.so $ROOT/paper_1501_04706_b200/csrc/{k_pre,k_rounds,k_gen,k_gather,seghull_b200,pts2_io,phases}.cu
