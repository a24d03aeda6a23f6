# quick GPU check: gpu tests, then bench lines for the configs given as arguments (c2 c3 c5 bf16)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for c in "$@"; do
  case $c in
    bf16) args="--precision bf16" ;;
    *) args="--config $c" ;;
  esac
  timeout 600 python bench.py --no-cpu $args > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - gpurun_out/bench_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d['roofline'].get('launch_us', {})
print(sys.argv[1], round(d['value']), {k: round(v, 1) for k, v in r.items()})
PY
done
