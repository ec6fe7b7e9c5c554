# ncu --set full of the gather kernel (96-camera C3 subset; plain run first)
mkdir -p gpurun_out
python tools/probe_matcher.py 96 0 > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:match_gather_kernel -s 1 -c 1 \
    -o gpurun_out/ga_prof -f python tools/probe_matcher.py 96 0 > gpurun_out/ncu_run.log 2>&1
echo "ncu rc=$?"
