# matcher A/B: parity tests of the matcher, then the C3 probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_guided_gpu.py tests/test_bench_parity_gpu.py tests/test_densify_gpu.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python tools/probe_matcher.py 320 0 > gpurun_out/ab_new.log 2>&1; echo "rc=$?" >> gpurun_out/ab_new.log
tail -3 gpurun_out/ab_tests.log; head -4 gpurun_out/ab_new.log
