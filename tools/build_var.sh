# build_var.sh NAME "-DFLAG ..." : a variant of the library into build_var/lib_NAME.so
mkdir -p build_var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off,-fopenmp -lgomp -I include -shared $2 -o build_var/lib_$1.so paper_1501_04706_b200/csrc/{k_pre,k_rounds,k_gen,seghull_b200,pts2_io}.cu
