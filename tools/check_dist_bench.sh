mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -x -q -m gpu > gpurun_out/dist_gpu.log 2>&1; echo "dist rc=$?" >> gpurun_out/dist_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
python bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_g2.log 2>&1; echo "g2 rc=$?" >> gpurun_out/bench_g2.log
tail -3 gpurun_out/dist_gpu.log; tail -c 1500 gpurun_out/bench_quick.log; cat gpurun_out/bench_g2.log
