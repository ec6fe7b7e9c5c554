# ncu --set full of the match kernel and the preparation kernels (96-camera C3 subset)
mkdir -p gpurun_out
python tools/probe_matcher.py 96 0 > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:match_ms_kernel -s 1 -c 1 \
    -o gpurun_out/ms_prof -f python tools/probe_matcher.py 96 0 > gpurun_out/ncu_run.log 2>&1
echo "ncu ms rc=$?"
ncu --set full --clock-control none --import-source on \
    -k 'regex:lines_kernel|groups_kernel|member_kernel|prep_kernel|sg_prep_kernel|scatter_kernel|sg_shape_kernel|compact_kernel' \
    -s 8 -c 8 -o gpurun_out/pre_prof -f python tools/probe_matcher.py 96 0 > gpurun_out/ncu_run2.log 2>&1
echo "ncu pre rc=$?"
