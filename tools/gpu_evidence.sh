# Round evidence on one B200: bench lines (C2 with CPU baseline, bf16, C3, C5), the C2
# launch list (cold-cache, serialised) and ncu --set full raw pages of one C2 forward and
# of the C3 dominant launch.  Usage: bash tools/gpu_evidence.sh TAG
tag=${1:-v}
o=gpurun_out
timeout 900 python bench.py > $o/bench_c2_$tag.json 2> $o/bench_c2_$tag.err
timeout 600 python bench.py --no-cpu --precision bf16 > $o/bench_bf16_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c3 > $o/bench_c3_$tag.json 2>&1
timeout 600 python bench.py --no-cpu --config c5 > $o/bench_c5_$tag.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o/launches_c2_$tag.csv python tools/prof_forward.py 128 64 2 > $o/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"tc_conv|gate_strips|head_strips|stem_const" \
  --launch-skip 13 --launch-count 13 -f -o /tmp/fwd python tools/prof_forward.py 128 64 2 > $o/ncu_fwd.log 2>&1
ncu -i /tmp/fwd.ncu-rep --page raw --csv > $o/fwd_raw_$tag.csv
timeout 900 ncu --set full --clock-control none -k regex:"head_tiles" --launch-skip 1 --launch-count 1 \
  -f -o /tmp/c3head python tools/prof_forward.py 256 1024 2 > $o/ncu_c3.log 2>&1
ncu -i /tmp/c3head.ncu-rep --page raw --csv > $o/c3head_raw_$tag.csv
for f in $o/bench_*_$tag.json; do tail -c 300 $f; echo; done
