# bench.py default workload, one line summary: value + per-launch kernel times
timeout 600 python bench.py --no-cpu $* > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/qb.json').read().strip().splitlines()[-1])
print(round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v, 1) for k, v in d['roofline']['launch_us'].items()})
PY
