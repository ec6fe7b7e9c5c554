# ncu --set full (source counters) of the current match kernel on the C3 bench step
mkdir -p gpurun_out
python tools/probe_matcher.py 320 0 > gpurun_out/nm_probe.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:match_ms_kernel -s 1 -c 1 \
      -o gpurun_out/nm_match -f python tools/probe_matcher.py 320 0 > gpurun_out/nm_ncu.log 2>&1; echo "ncu match rc=$?"
