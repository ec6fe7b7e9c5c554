mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/all_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/all_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
tail -4 gpurun_out/all_gpu.log; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_quick.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); L=d.get('localization',{})
    print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])
    print('loc', L.get('value'), L.get('e2e',{}).get('value'), L.get('status_counts'), L.get('roofline',{}).get('frac'))
else:
    print(open('gpurun_out/bench_quick.log').read()[-3000:])
PY
