# Round-2 measurement set: bench (b200 + reference arms), the bench's launch list,
# and ncu --set full captures of the three dominant kernels.  Each ncu command runs
# only after the same program exited 0 without ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02_smi.txt
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 1500 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu \
      > gpurun_out/r02_ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/probe_matcher.py 320 0 > gpurun_out/r02_probe_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:match_ms_kernel -s 1 -c 1 \
      -o gpurun_out/r02_match -f python tools/probe_matcher.py 320 0 > gpurun_out/r02_ncu_match.log 2>&1; echo "ncu match rc=$?"
ncu --set full --clock-control none --import-source on -k regex:setup_kernel -s 1 -c 1 \
    -o gpurun_out/r02_setup -f python tools/probe_matcher.py 320 0 > gpurun_out/r02_ncu_setup.log 2>&1; echo "ncu setup rc=$?"
python tools/probe_knn.py > gpurun_out/r02_probe_knn.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:knn_tc_kernel -s 2 -c 1 \
      -o gpurun_out/r02_knn -f python tools/probe_knn.py > gpurun_out/r02_ncu_knn.log 2>&1; echo "ncu knn rc=$?"
