# Round-2 evidence on one B200: bench lines of every config (C2 with the CPU baseline), the
# reference arm, the C1 latency line, and the C2 launch list.  Usage: bash tools/gpu_evidence_r2.sh TAG
tag=${1:-v}
o=gpurun_out
timeout 900 python bench.py > $o/r2_bench_c2_$tag.json 2> $o/r2_bench_c2_$tag.err
timeout 600 python bench.py --no-cpu --precision bf16 > $o/r2_bench_bf16_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c3 > $o/r2_bench_c3_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c3 --precision bf16 > $o/r2_bench_c3bf16_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c4 > $o/r2_bench_c4_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c5 > $o/r2_bench_c5_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c1 > $o/r2_bench_c1_$tag.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/r2_bench_ref_$tag.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o/r2_launches_c2_$tag.csv python tools/prof_forward.py 128 64 2 > $o/ncu_launch.log 2>&1
for f in $o/r2_bench_*_$tag.json; do echo "$f"; tail -c 400 $f; echo; done
