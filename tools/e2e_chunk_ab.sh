# e2e (host-buffer API) throughput per config; args = STDA_HOST_CHUNK_MB values (0 = default rule)
for mb in "$@"; do for c in c2 c3 c5; do
  env $( [ "$mb" != 0 ] && echo STDA_HOST_CHUNK_MB=$mb ) python bench.py --no-cpu --config $c 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mb', '$c', round(d['value']), round(d['e2e']['value']))"
done; done
