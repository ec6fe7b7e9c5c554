mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_coarse_gpu.py -x -q -m gpu > gpurun_out/fund.log 2>&1; echo "rc=$?" >> gpurun_out/fund.log
bash tools/run_ref_under_install.sh > /dev/null 2>&1
tail -3 gpurun_out/fund.log; tail -4 gpurun_out/ref_under_install.log
