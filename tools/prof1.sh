o=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"tc_conv_kernel" --launch-skip 9 --launch-count 1 -f -o /tmp/stemt python tools/prof_forward.py 128 64 2 > $o/ncu_stemt.log 2>&1
ncu -i /tmp/stemt.ncu-rep --page raw --csv > $o/stemt_raw.csv
python tools/ncu_brief.py $o/stemt_raw.csv > $o/stemt_brief.txt
ncu -i /tmp/stemt.ncu-rep --page source --csv --print-source sass > /tmp/stemt_src.csv
python tools/ncu_stalls.py /tmp/stemt_src.csv 30 > $o/stemt_stalls.txt 2>&1
