mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
bash tools/check_all.sh > gpurun_out/check_all.txt 2>&1
timeout 300 python tools/probe_matcher.py 320 0 > gpurun_out/probe_c3.log 2>&1
