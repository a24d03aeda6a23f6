# Round evidence: CTA timelines, the C2 launch list and one ncu --set full capture of a C2
# forward (raw page + per-kernel source-page stall summaries).  Usage: bash tools/gpu_profile.sh TAG
tag=${1:-v}
o=gpurun_out
timeout 300 python tools/tc_trace.py 128 128 64 fp32 > $o/trace_$tag.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o/launches_c2_$tag.csv python tools/prof_forward.py 128 64 2 > $o/ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"tc_conv|gate_strips|head_strips|stem_" --launch-skip 13 --launch-count 13 -f -o /tmp/fwd_$tag \
  python tools/prof_forward.py 128 64 2 > $o/ncu_fwd.log 2>&1
ncu -i /tmp/fwd_$tag.ncu-rep --page raw --csv > $o/fwd_raw_$tag.csv
python tools/ncu_brief.py $o/fwd_raw_$tag.csv > $o/fwd_brief_$tag.txt
for i in 0 1 2 3 4 5 6 7 8 9 10 11 12; do
  ncu -i /tmp/fwd_$tag.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 \
    > /tmp/src_$i.csv 2>/dev/null && python tools/ncu_stalls.py /tmp/src_$i.csv 12 > $o/stalls_${tag}_$i.txt 2>&1
done
