# e2e (host-buffer API) of bench.py's default workload under env switches: bash tools/e2e_ab.sh "X=0" "A=1 B=2" ...
for envs in "$@"; do
  env $envs timeout 300 python bench.py --no-cpu --steps 20 ${AB_ARGS:-} > gpurun_out/e2e_tmp.json 2>/dev/null
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/e2e_tmp.json').read().strip().splitlines()[-1])
print(sys.argv[1], 'value', round(d['value']), 'e2e', round(d['e2e']['value']), [round(c) for c in d['e2e']['calls']])
PY
done
