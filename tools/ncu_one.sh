# ncu --set full of ONE launch of a C2 forward: bash tools/ncu_one.sh KERNEL_REGEX LAUNCH_SKIP TAG [hw B]
# -> gpurun_out/<TAG>_brief.txt (counters) and <TAG>_stalls.txt (source-level stall sites)
re=$1; skip=$2; tag=$3; hw=${4:-128}; B=${5:-64}
o=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$re" --launch-skip $skip --launch-count 1 \
  -f -o /tmp/$tag python tools/prof_forward.py $hw $B 2 > $o/ncu_$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv > $o/${tag}_raw.csv
python tools/ncu_brief.py $o/${tag}_raw.csv > $o/${tag}_brief.txt
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > /tmp/${tag}_src.csv
python tools/ncu_stalls.py /tmp/${tag}_src.csv 30 > $o/${tag}_stalls.txt 2>&1
