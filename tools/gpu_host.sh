# host-overhead A/B: bare C call and the Python API per library variant, then the GPU test suite
for v in build_var/*.so; do echo "== $v"; SHB_LIB=$v python tools/py_overhead.py; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest.log
