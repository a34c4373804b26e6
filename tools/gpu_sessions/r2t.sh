O=gpurun_out/r2t; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 ./build/cpp/test_lsapgpu > $O/cpp_test.log 2>&1; echo "rc=$?" >> $O/cpp_test.log
