# Round-2 final measurement set (the reference arm's code path is unchanged since
# profiles/r02_bench_reference.json): ncu captures of the match / setup kernels
# (each after the same program exited 0 without ncu), their summaries, the bench
# (which reads the refreshed match summary), the bench's launch list and the launch
# list of one resident C3 step.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02f_smi.txt
python tools/probe_matcher.py 320 0 > gpurun_out/r02f_probe_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:match_ms_kernel -s 1 -c 1 \
      -o gpurun_out/r02f_match -f python tools/probe_matcher.py 320 0 > gpurun_out/r02f_ncu_match.log 2>&1; echo "ncu match rc=$?"
ncu --set full --clock-control none --import-source on -k regex:setup_kernel -s 1 -c 1 \
    -o gpurun_out/r02f_setup -f python tools/probe_matcher.py 320 0 > gpurun_out/r02f_ncu_setup.log 2>&1; echo "ncu setup rc=$?"
python tools/ncu_summary.py gpurun_out/r02f_match.ncu-rep gpurun_out/r02f_ncu_match_kernel.json 5401 > /dev/null && \
  cp gpurun_out/r02f_ncu_match_kernel.json profiles/ncu_match_kernel.json
python tools/ncu_summary.py gpurun_out/r02f_setup.ncu-rep gpurun_out/r02f_ncu_setup_kernel.json 5401 > /dev/null
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02f_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu \
      > gpurun_out/r02f_ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/one_step.py > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(plan|setup|match|compact)' -s 8 --csv \
      --log-file gpurun_out/r02f_one_step_launches.csv python tools/one_step.py > gpurun_out/r02f_one_step.log 2>&1; echo "one step rc=$?"
