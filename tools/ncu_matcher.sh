# ncu --set full of the match kernel on a C3-recipe subset (96 cameras); plain run first.
mkdir -p gpurun_out
K=${1:-match_team_kernel}
python tools/probe_matcher.py 96 0 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/ms_prof -f python tools/probe_matcher.py 96 0 > gpurun_out/ncu_run.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_run.log; head -3 gpurun_out/ncu_plain.log
