# CTA-0 timeline of the first tensor-core launch (the stem) under the epilogue ablations
for dbg in 0 1 2 8; do
  echo "=== STDA_TC_DBG=$dbg"
  STDA_TC_DBG=$dbg timeout 300 python tools/tc_trace.py 128 128 64 fp32 2>&1 | sed -n 1,6p
done
