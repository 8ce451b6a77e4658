#!/bin/bash
# ab_bench.sh -- measurement tool: interleaved bench runs of several builds of
# the library (OMPDS_LIB_PATH) on one box, so box-to-box variation cancels.
#   tools/ab_bench.sh lib1.so lib2.so ...   (on the GPU box)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in "$@"; do
    OMPDS_LIB_PATH=$lib python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['configs']
print('%-40s stream %7.1f GB/s  cfg1 %6.1f ns  cfg2 %7.1f GB/s  cfg3 %7.1f ns  agg %5.2f G/s  handle %5.1f us  sm %s' % ('$lib', d['value'], d['regions']['ns_per_region'], c['config2_shared_array']['GBps'], c['config3_nested_1team']['ns_per_region'], d['regions']['aggregate_regions_per_s'] / 1e9, d['regions']['team_handle_us_per_call'], d['clocks']['sm_mhz']))"
  done
done
