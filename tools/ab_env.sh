#!/bin/bash
# A/B timing of engine env switches: each argument is one run's env assignments
# ("X=0" for the default), e.g.  bash tools/ab_env.sh X=0 "STDA_TC_TSTAGES=4"
# prints triplets/s and the per-launch device times of bench.py's default workload.
for envs in "$@"; do
  env $envs python bench.py --steps 200 ${AB_ARGS:-} > /tmp/ab_tmp.json 2>/dev/null
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open('/tmp/ab_tmp.json').read().strip().splitlines()[-1])
r = d['roofline']['launch_us']
print(sys.argv[1], round(d['value']), {k: round(v, 1) for k, v in r.items()})
PY
done
