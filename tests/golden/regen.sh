#!/usr/bin/env bash
# Regenerates the golden vectors in this directory from the UNMODIFIED
# reference (compiled in place by oracle/Makefile; needs /root/reference).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(cd "$here/../.." && pwd)"
make -C "$repo/oracle" ref
"$repo/oracle/_ref/ref_golden" /root/reference/proj "$here"
