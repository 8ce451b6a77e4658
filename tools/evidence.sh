#!/bin/bash
# evidence.sh TAG -- one GPU call that refreshes the judged evidence for the
# current build: GPU tests + smoke, the bench line and the reference arm,
# ncu captures of every config kernel + the bench launch list
# (tools/ncu_capture_r2.sh), compute-sanitizer (tools/sanitize_all.sh).
# Everything lands in gpurun_out/TAG* (summarised into profiles/ afterwards).
cd "$(dirname "$0")/.."
tag=${1:-r2}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 1800 bash tools/ncu_capture_r2.sh $out/ncu > $out/ncu_capture.log 2>&1
# DRAM traffic of this build's bench kernel, for the bench line's roofline.traffic
python tools/ncu_summary.py --rep $out/ncu/stream.ncu-rep --name ${tag}_stream_ncu \
  --algo-bytes 6442450944 --traffic-n 268435456 > /dev/null && cp profiles/traffic.json $out/
sleep 2
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference > $out/reference_arm.json 2> $out/reference_arm.err
timeout 3000 bash tools/sanitize_all.sh $tag > $out/sanitize.log 2>&1
tail -2 $out/gpu_tests.log; cat $out/smoke.log | tail -1; cat $out/sanitize.log
