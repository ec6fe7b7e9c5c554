# int8 tcgen05 and FP64 peaks on the box -> profiles/measured_peaks_extra.json
# (tools/bin/peaks is built here: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/peaks tools/peaks.cu)
mkdir -p gpurun_out
test -x tools/bin/peaks && \
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
timeout 120 tools/bin/peaks > gpurun_out/peaks.json 2>&1; echo "rc=$?" >> gpurun_out/peaks.log
kill $SMI 2>/dev/null
cat gpurun_out/peaks.json; tail -5 gpurun_out/peaks_clocks.csv
