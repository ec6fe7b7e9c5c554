# A/B of the match kernels: parity tests on the new kernel, then the C3 probe for both.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_guided_gpu.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python tools/probe_matcher.py 320 0 > gpurun_out/ab_new.log 2>&1; echo "rc=$?" >> gpurun_out/ab_new.log
MSFM_MATCH_V1=1 timeout 300 python tools/probe_matcher.py 320 0 > gpurun_out/ab_v1.log 2>&1; echo "rc=$?" >> gpurun_out/ab_v1.log
tail -5 gpurun_out/ab_tests.log; cat gpurun_out/ab_new.log gpurun_out/ab_v1.log
