# C1 (batch-1) latency under engine env switches: bash tools/c1_ab.sh "X=0" "STDA_PDL=1" ...
for envs in "$@"; do
  env $envs timeout 300 python bench.py --no-cpu --config c1 > gpurun_out/c1_tmp.json 2>/dev/null
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/c1_tmp.json').read().strip().splitlines()[-1])
l = d['latency']
print(sys.argv[1], 'graph p50', round(l['graph_replay']['p50_us'], 1), 'eager p50', round(l['eager_forward']['p50_us'], 1),
      'host p50', round(l['host_buffers']['p50_us'], 1), 'step_ms', round(d['ms_per_step'] * 1e3, 1))
PY
done
