# ncu --set full of the matcher's preparation kernels (96-camera C3 subset; plain run first)
mkdir -p gpurun_out
python tools/probe_matcher.py 96 0 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k 'regex:lines_kernel|groups_kernel|member_kernel|prep_kernel|sg_prep_kernel|scatter_kernel|sg_shape_kernel|compact_kernel' \
    -s 8 -c 8 -o gpurun_out/pre_prof -f python tools/probe_matcher.py 96 0 > gpurun_out/ncu_run.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_run.log
