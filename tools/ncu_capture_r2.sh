#!/usr/bin/env bash
# Round-2 ncu captures (one GPU): --set full of each config kernel, the
# launch list of a bench run, and the SASS of the built library.
set -x
out=${1:-gpurun_out/r2}
mkdir -p $out
K1='regex:.*RegionsProg.*'; K2='regex:.*SharedArrayProg.*'; K3='regex:.*NestedProg.*'; K4='regex:.*StreamProg.*'
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
$NCU -k "$K1" -s 1 -c 1 -o $out/regions -f python tools/regions_long_probe.py > $out/regions.log 2>&1
$NCU -k "$K1" -s 1 -c 1 -o $out/regions_full -f python tools/regions_full_probe.py > $out/regions_full.log 2>&1
$NCU -k "$K2" -s 1 -c 1 -o $out/config2 -f python tools/config2_probe.py > $out/config2.log 2>&1
$NCU -k "$K3" -s 1 -c 1 -o $out/nested -f python tools/nested_full_probe.py > $out/nested.log 2>&1
$NCU -k "$K4" -s 2 -c 1 -o $out/stream -f python bench.py --steps 3 --warmup 3 --only-stream --no-e2e --no-cpu > $out/stream.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > $out/launch_bench.log 2>&1
ls -la $out
