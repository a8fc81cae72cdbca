#!/bin/bash
# Bench the product .so and each variant .so named on the command line (GPU box).
# usage: tools/variants.sh [variant ...]   (variant = name under paper_2511_00292_b200/build/variants)
for v in "" "$@"; do
  so=""; [ -n "$v" ] && so=$PWD/paper_2511_00292_b200/build/variants/$v.so
  printf "%-12s " "${v:-product}"
  EIG33_SO=$so timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --no-multi-driver 2>&1 | python -c "
import json,sys
l=sys.stdin.read().strip().splitlines()
try:
  d=json.loads(l[-1]); c=d['clocks']
  print('%.2f G/s  %.3f ms  frac %.3f  sm %s MHz %s' % (d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], c['sm_mhz'], c['reasons']))
except Exception as e:
  print('FAILED', l[-3:])"
done
