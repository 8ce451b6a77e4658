#!/bin/bash
# region_variants.sh -- measurement tool (not product): builds
# tools/latency_ladder.cu once per device-runtime option set and runs each,
# so the marginal cost of every protocol optimisation of the config-1 region
# is measured on the same box in one call.
#
#   tools/region_variants.sh build   # here (nvcc cross-compiles)
#   tools/region_variants.sh run     # on the GPU box
set -e
cd "$(dirname "$0")/.."
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
declare -A V
V[base]="-DOMPDS_PREFETCH_WINDOW=0 -DOMPDS_SOLE_WARP_RETIRE=0"
V[prefetch]="-DOMPDS_PREFETCH_WINDOW=1 -DOMPDS_SOLE_WARP_RETIRE=0"
V[sole]="-DOMPDS_PREFETCH_WINDOW=0 -DOMPDS_SOLE_WARP_RETIRE=1"
V[all]=""
ORDER="base prefetch sole all"
case "$1" in
build)
  for k in $ORDER; do
    $NVCC -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ${V[$k]} \
      -I paper_1711_10413_b200/csrc tools/latency_ladder.cu \
      paper_1711_10413_b200/csrc/ompds_host.cpp -o tools/ladder_$k.bin 2>/dev/null &
  done
  wait
  ls -la tools/ladder_*.bin
  ;;
run)
  for k in $ORDER; do
    echo "== $k: ${V[$k]}"
    timeout 60 tools/ladder_$k.bin
  done
  ;;
*)
  echo "usage: $0 build|run" >&2
  exit 2
  ;;
esac
