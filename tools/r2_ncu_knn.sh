mkdir -p gpurun_out
python tools/probe_knn.py > gpurun_out/knn_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:knn_tc_kernel -s 2 -c 1 \
    -o gpurun_out/knn_prof -f python tools/probe_knn.py > gpurun_out/ncu_knn_run.log 2>&1
echo "ncu rc=$?"
