mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_localize_gpu.py tests/test_descriptors.py tests/test_coarse_gpu.py -x -q -m gpu > gpurun_out/knn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/knn_tests.log
tail -15 gpurun_out/knn_tests.log
