#!/bin/bash
# ab_cfg1.sh -- measurement tool: interleaved config-1 sweeps (tools/cfg1_sweep.py)
# and bench lines (tools/ab_bench.sh) of several library builds on one box.
#   tools/ab_cfg1.sh OUTDIR lib1.so lib2.so ...   (on the GPU box)
cd "$(dirname "$0")/.."
out=$1; shift
mkdir -p $out
for rep in 1 2; do
  for lib in "$@"; do
    v=$(basename $lib .so)
    OMPDS_LIB_PATH=$lib PER_SM=${PER_SM:-16,20,22,24,28,32} timeout 300 \
      python tools/cfg1_sweep.py $out/cfg1_${v}_${rep}.json > /dev/null 2>&1
  done
done
timeout 900 bash tools/ab_bench.sh "$@" > $out/ab_bench.txt 2>&1
python - "$out" <<'PY'
import glob, json, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "cfg1_*.json"))):
    d = json.load(open(f))
    agg = {k: round(v / 1e9, 2) for k, v in d["regions_per_s_by_teams_per_sm"].items()}
    print(os.path.basename(f), round(d["ns_per_region_1team_torch.int32"], 1),
          round(d["ns_per_region_1team_torch.float64"], 1), agg)
PY
